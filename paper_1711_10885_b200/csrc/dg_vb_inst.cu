// One translation unit per (n, m) of the variable-velocity / over-integrated kernel
// (dg_vb.cuh; compiled with -DDG_N=n -DDG_M=m): table upload, launcher, launch facts.
#include "dg_vb.cuh"

#define DG_CAT3_(a, b, c, d) a##b##_##c##d
#define DG_CAT3(a, b, c, d) DG_CAT3_(a, b, c, d)

namespace dg {

template <int N, int M>
static void fill_eo_m(EO<M>& o, const double (&A)[MMAX][MMAX], bool transpose)
{
    constexpr int H = M / 2;
    auto a = [&](int i, int j) { return transpose ? A[j][i] : A[i][j]; };
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < H; ++j) {
            o.p[i][j] = 0.5 * (a(i, j) + a(i, M - 1 - j));
            o.m[i][j] = 0.5 * (a(i, j) - a(i, M - 1 - j));
        }
    for (int i = 0; i < H; ++i) {
        o.col[i] = (M & 1) ? a(i, H) : 0.0;
        o.row[i] = (M & 1) ? a(H, i) : 0.0;
    }
}

int DG_CAT3(upload_tables_vb_n, DG_N, m, DG_M)(const HostTables& t)
{
    constexpr int N = DG_N, M = DG_M;
    if (t.n != N || t.m != M) return -1;
    static vb::TabV<N, M> h;
    for (int c = 0; c < 6; ++c)
        for (int i = 0; i < vb::TabV<N, M>::HM; ++i)
            for (int j = 0; j < N; ++j) h.Vh[c][i][j] = t.V[i][j];
    for (int c = 0; c < 3; ++c) {
        fill_eo_m<N, M>(h.Dc[c], t.Dc, false);
        fill_eo_m<N, M>(h.DcT[c], t.Dc, true);
    }
    for (int i = 0; i < M; ++i) {
        h.w[i] = t.w[i];
        h.xi[i] = t.xi[i];
        for (int c = 0; c < 3; ++c) {
            h.L[c][0][i] = t.L0[i];
            h.L[c][1][i] = t.L1[i];
            h.L[c][2][i] = t.LD0[i];
            h.L[c][3][i] = t.LD1[i];
        }
    }
    for (int j = 0; j < N; ++j) {
        h.th0[j] = t.th0[j];
        h.th1[j] = t.th1[j];
        h.dth0[j] = t.dth0[j];
        h.dth1[j] = t.dth1[j];
    }
    return cudaMemcpyToSymbol(vb::g_tabv, &h, sizeof(h)) == cudaSuccess ? 0 : -3;
}

static int g_attr[64];

cudaError_t DG_CAT3(launch_vb_n, DG_N, m, DG_M)(const KParams& p, cudaStream_t s)
{
    constexpr int N = DG_N, M = DG_M;
    if (p.ntasks <= 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !g_attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(vb::dg_vb_kernel<N, M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             vb::VSmem<N, M>::BYTES);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(vb::dg_vb_kernel<N, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     vb::VSmem<N, M>::BYTES);
        if (e != cudaSuccess) return e;
        g_attr[dev] = 1;
    }
    constexpr int C = vb::VCfg<M>::C;
    const unsigned grid = (unsigned)((p.ntasks + C - 1) / C);
    if (p.ghosts) vb::dg_vb_kernel<N, M, true><<<grid, vb::VCfg<M>::TPC, vb::VSmem<N, M>::BYTES, s>>>(p);
    else vb::dg_vb_kernel<N, M, false><<<grid, vb::VCfg<M>::TPC, vb::VSmem<N, M>::BYTES, s>>>(p);
    return cudaGetLastError();
}

int DG_CAT3(vb_info_n, DG_N, m, DG_M)(LaunchInfo* info)
{
    constexpr int N = DG_N, M = DG_M;
    info->cells_per_cta = vb::VCfg<M>::C;
    info->threads = vb::VCfg<M>::TPC;
    info->smem = vb::VSmem<N, M>::BYTES;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, vb::dg_vb_kernel<N, M, false>) != cudaSuccess) return -3;
    info->regs = fa.numRegs;
    if (cudaFuncSetAttribute(vb::dg_vb_kernel<N, M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             vb::VSmem<N, M>::BYTES) != cudaSuccess)
        return -3;
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, vb::dg_vb_kernel<N, M, false>, info->threads,
                                                      vb::VSmem<N, M>::BYTES) != cudaSuccess)
        return -3;
    info->ctas_per_sm = blocks;
    return 0;
}

}  // namespace dg
