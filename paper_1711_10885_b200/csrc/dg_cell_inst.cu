// One translation unit per basis size n = k+1 (compiled with -DDG_N=n): the
// fused cell kernel instantiation, its __constant__ table upload and launcher.
#include "dg_cell.cuh"

#include <cstring>

#define DG_CAT2(a, b) a##b
#define DG_CAT(a, b) DG_CAT2(a, b)

namespace dg {

template <int N>
static void fill_eo(EO<N>& o, const double (&A)[NMAX][NMAX], bool transpose)
{
    constexpr int H = N / 2;
    auto a = [&](int i, int j) { return transpose ? A[j][i] : A[i][j]; };
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < H; ++j) {
            o.p[i][j] = 0.5 * (a(i, j) + a(i, N - 1 - j));
            o.m[i][j] = 0.5 * (a(i, j) - a(i, N - 1 - j));
        }
    for (int i = 0; i < H; ++i) {
        o.col[i] = (N & 1) ? a(i, H) : 0.0;
        o.row[i] = (N & 1) ? a(H, i) : 0.0;
    }
}

int DG_CAT(upload_tables_n, DG_N)(const HostTables& t)
{
    constexpr int N = DG_N;
    if (t.n != N) return -1;
    static Tab<N> h;
    for (int c = 0; c < 12; ++c)
        for (int i = 0; i < Tab<N>::HC; ++i)
            for (int j = 0; j < N; ++j) h.Vh[c][i][j] = t.V[i][j];
    for (int c = 0; c < 6; ++c) {
        fill_eo<N>(h.Dc[c], t.Dc, false);
        fill_eo<N>(h.DcT[c], t.Dc, true);
    }
    for (int i = 0; i < N; ++i) {
        h.w[i] = t.w[i];
        for (int c = 0; c < 6; ++c) {
            h.L[c][0][i] = t.L0[i];
            h.L[c][1][i] = t.L1[i];
            h.L[c][2][i] = t.LD0[i];
            h.L[c][3][i] = t.LD1[i];
        }
        h.th0[i] = t.th0[i];
        h.th1[i] = t.th1[i];
        h.dth0[i] = t.dth0[i];
        h.dth1[i] = t.dth1[i];
    }
    return cudaMemcpyToSymbol(g_tab, &h, sizeof(h)) == cudaSuccess ? 0 : -3;
}

static int g_attr_done[64];

cudaError_t DG_CAT(launch_cell_n, DG_N)(const KParams& p, cudaStream_t s)
{
    constexpr int N = DG_N;
    constexpr int C = Cfg<N>::C;
    constexpr int THREADS = C * Cfg<N>::TPC;
    if (p.ntasks <= 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !g_attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(dg_cell_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Smem<N>::BYTES);
        if (e != cudaSuccess) return e;
        g_attr_done[dev] = 1;
    }
    const int64_t grid = (p.ntasks + C - 1) / C;
    dg_cell_kernel<N><<<(unsigned)grid, THREADS, Smem<N>::BYTES, s>>>(p);
    return cudaGetLastError();
}

int DG_CAT(cell_info_n, DG_N)(LaunchInfo* info)
{
    constexpr int N = DG_N;
    info->cells_per_cta = Cfg<N>::C;
    info->threads = Cfg<N>::C * Cfg<N>::TPC;
    info->smem = Smem<N>::BYTES;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, dg_cell_kernel<N>) != cudaSuccess) return -3;
    info->regs = fa.numRegs;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !g_attr_done[dev]) {
        if (cudaFuncSetAttribute(dg_cell_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<N>::BYTES) !=
            cudaSuccess)
            return -3;
        g_attr_done[dev] = 1;
    }
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, dg_cell_kernel<N>, info->threads, Smem<N>::BYTES) !=
        cudaSuccess)
        return -3;
    info->ctas_per_sm = blocks;
    return 0;
}

}  // namespace dg
