// One translation unit per basis size n = k+1 (compiled with -DDG_N=n): the
// fused cell kernel instantiation, its __constant__ table upload and launcher.
#include "dg_cell.cuh"
#include "dg_gen.cuh"
#include "dg_reg.cuh"
#if DG_N == 8
#include "dg_mma8.cuh"
#endif

#include <cstdlib>
#include <cstring>

#define DG_CAT2(a, b) a##b
#define DG_CAT(a, b) DG_CAT2(a, b)

namespace dg {

template <int N>
static void fill_eo(EO<N>& o, const double (&A)[MMAX][MMAX], bool transpose)
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
    {   // sigma/delta form (dg_cell.cuh): doubled forward V, doubled Dc and Dc^T diag(w)
        static double D2[MMAX][MMAX], A2[MMAX][MMAX];
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                D2[i][j] = 2.0 * t.Dc[i][j];
                A2[i][j] = 2.0 * t.Dc[j][i] * t.w[j];
            }
        for (int c = 0; c < 9; ++c)
            for (int i = 0; i < Tab<N>::HC; ++i)
                for (int j = 0; j < N; ++j) h.Vs[c][i][j] = ((N & 1) && i == N / 2 ? 1.0 : 2.0) * t.V[i][j];
        for (int c = 0; c < 3; ++c) {
            fill_eo<N>(h.DcTws[c], A2, false);
            for (int i = 0; i < N / 2; ++i) h.DcTws[c].row[i] *= 0.5;   // the middle row (odd n) stays plain
        }
        for (int c = 0; c < 5; ++c) {
            fill_eo<N>(h.Dcs[c], D2, false);
            fill_eo<N>(h.DcTs[c], D2, true);
            for (int i = 0; i < N / 2; ++i) {
                h.Dcs[c].row[i] *= 0.5;
                h.DcTs[c].row[i] *= 0.5;
            }
        }
        constexpr int H = N / 2;
        for (int i = 0; i < Tab<N>::HC; ++i)
            for (int j = 0; j < N; ++j) h.Gs[i][j] = ((N & 1) && i == H ? 1.0 : 2.0) * t.G[i][j];
        const double* rows[4] = {t.L0, t.L1, t.LD0, t.LD1};
        for (int r = 0; r < 4; ++r) {
            const double* l = rows[r];
            for (int i = 0; i < H; ++i) {
                for (int c = 0; c < 2; ++c) {
                    h.Ls[c][r][i] = 0.5 * (l[i] + l[N - 1 - i]);
                    h.Ls[c][r][N - 1 - i] = 0.5 * (l[i] - l[N - 1 - i]);
                }
                h.Lsl[r][i] = l[i] + l[N - 1 - i];
                h.Lsl[r][N - 1 - i] = l[i] - l[N - 1 - i];
            }
            if (N & 1) {
                h.Ls[0][r][H] = h.Ls[1][r][H] = l[H];
                h.Lsl[r][H] = l[H];
            }
        }
    }
    {
        constexpr int H = N / 2;
        for (int c = 0; c < 3; ++c) {
            for (int i = 0; i < H; ++i) {
                h.Le[c][0][i] = 0.5 * (t.L0[i] + t.L0[N - 1 - i]);
                h.Le[c][1][i] = 0.5 * (t.L0[i] - t.L0[N - 1 - i]);
                h.Le[c][2][i] = 0.5 * (t.LD0[i] + t.LD0[N - 1 - i]);
                h.Le[c][3][i] = 0.5 * (t.LD0[i] - t.LD0[N - 1 - i]);
            }
            h.Lmid[c][0] = (N & 1) ? t.L0[H] : 0.0;
            h.Lmid[c][1] = (N & 1) ? t.LD0[H] : 0.0;
        }
    }
    for (int i = 0; i < N; ++i) {
        h.w[i] = t.w[i];
        h.th0[i] = t.th0[i];
        h.th1[i] = t.th1[i];
        h.dth0[i] = t.dth0[i];
        h.dth1[i] = t.dth1[i];
    }
    if (cudaMemcpyToSymbol(g_tab, &h, sizeof(h)) != cudaSuccess) return -3;
    {
        static RTab<N> rt;
        for (int i = 0; i < N; ++i) {
            for (int j = 0; j < N; ++j) {
                rt.V[i][j] = t.V[i][j];
                rt.G[i][j] = t.G[i][j];
                rt.Dc[i][j] = t.Dc[i][j];
            }
            rt.w[i] = t.w[i];
            rt.L[0][i] = t.L0[i];
            rt.L[1][i] = t.L1[i];
            rt.L[2][i] = t.LD0[i];
            rt.L[3][i] = t.LD1[i];
            rt.th0[i] = t.th0[i];
            rt.th1[i] = t.th1[i];
            rt.dth0[i] = t.dth0[i];
            rt.dth1[i] = t.dth1[i];
        }
        if (cudaMemcpyToSymbol(g_rtab, &rt, sizeof(rt)) != cudaSuccess) return -3;
    }
#if DG_N == 8
    // per-lane DMMA fragments (dg_mma8.cuh): lane l -> g = l >> 2, t = l & 3
    static double fr[32][16];
    auto Lm = [&](int i, int r) { return r == 0 ? t.L0[i] : r == 1 ? t.L1[i] : r == 2 ? t.LD0[i] : r == 3 ? t.LD1[i] : 0.0; };
    for (int l = 0; l < 32; ++l) {
        const int g = l >> 2, tt = l & 3;
        for (int c = 0; c < 2; ++c) {
            fr[l][m8::F_VF0 + c] = t.V[g][2 * tt + c];
            fr[l][m8::F_VB0 + c] = t.V[2 * tt + c][g];
            fr[l][m8::F_DC0 + c] = t.Dc[g][2 * tt + c];
            fr[l][m8::F_DT0 + c] = t.Dc[2 * tt + c][g];
            fr[l][m8::F_LT0 + c] = Lm(2 * tt + c, g);
            fr[l][m8::F_WT0 + c] = t.w[2 * tt + c];
        }
        fr[l][m8::F_LL] = Lm(g, tt);
        fr[l][m8::F_WG] = t.w[g];
        for (int k = m8::F_COUNT; k < 16; ++k) fr[l][k] = 0.0;
    }
    if (cudaMemcpyToSymbol(m8::g_frag, fr, sizeof(fr)) != cudaSuccess) return -3;
#endif
    return 0;
}

// n = 8: the DMMA kernel with DG_CELL_KERNEL=mma (default: the SIMT kernel while it is faster)
static bool use_mma()
{
#if DG_N == 8
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("DG_CELL_KERNEL");
        v = (e && std::strcmp(e, "mma") == 0) ? 1 : 0;
    }
    return v == 1;
#else
    return false;
#endif
}

static int g_attr_done[64];

// n <= DG_REG_NMAX: the register-resident kernel (dg_reg.cuh) unless DG_CELL_KERNEL=pencil
static bool use_reg()
{
    if (DG_N > DG_REG_NMAX) return false;
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("DG_CELL_KERNEL");
        v = (e && std::strcmp(e, "pencil") == 0) ? 0 : 1;
    }
    return v == 1;
}
constexpr int REG_THREADS = REG_CTA;
// dynamic shared memory of the register kernel (the staged images, RStage; 0 when not staged)
template <int N, bool GEN, bool GH>
static cudaError_t reg_attr()
{
    static int done[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (RStage<N, GEN>::BYTES == 0 || dev < 0 || dev >= 64 || done[dev]) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(dg_reg_kernel<N, GEN, GH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         RStage<N, GEN>::BYTES);
    if (e == cudaSuccess) done[dev] = 1;
    return e;
}

cudaError_t DG_CAT(launch_cell_n, DG_N)(const KParams& p, cudaStream_t s)
{
    constexpr int N = DG_N;
    constexpr int C = Cfg<N>::C;
    constexpr int THREADS = C * Cfg<N>::TPC;
    if (p.ntasks <= 0) return cudaSuccess;
    if constexpr (N <= DG_REG_NMAX) {
        if (use_reg()) {
            const int64_t grid = (p.ntasks + REG_THREADS - 1) / REG_THREADS;
            if (p.ghosts) { cudaError_t e = reg_attr<N, false, true>(); if (e != cudaSuccess) return e; dg_reg_kernel<N, false, true><<<(unsigned)grid, REG_THREADS, RStage<N, false>::BYTES, s>>>(p); }
            else { cudaError_t e = reg_attr<N, false, false>(); if (e != cudaSuccess) return e; dg_reg_kernel<N, false, false><<<(unsigned)grid, REG_THREADS, RStage<N, false>::BYTES, s>>>(p); }
            return cudaGetLastError();
        }
    }
    int dev = 0;
    cudaGetDevice(&dev);
#if DG_N == 8
    bool ghosts = false;
    for (int f = 0; f < 6; ++f) ghosts = ghosts || p.ghost[f] != nullptr;
    // DMMA variant: no wrap, no SSP epilogue, single rank (it reads neighbours as blocks, not traces)
    if (use_mma() && !(p.per[0] | p.per[1] | p.per[2]) && p.epi != 2 && !ghosts) {
        static int done[64];
        constexpr int BYTES = m8::C * m8::PER_CELL * 8;
        if (dev >= 0 && dev < 64 && !done[dev]) {
            cudaError_t e = cudaFuncSetAttribute(m8::dg_cell_mma8, cudaFuncAttributeMaxDynamicSharedMemorySize, BYTES);
            if (e != cudaSuccess) return e;
            done[dev] = 1;
        }
        const int64_t grid = (p.ntasks + m8::C - 1) / m8::C;
        m8::dg_cell_mma8<<<(unsigned)grid, 32 * m8::C, BYTES, s>>>(p);
        return cudaGetLastError();
    }
#endif
    if (dev >= 0 && dev < 64 && !g_attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(dg_cell_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Smem<N>::BYTES);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(dg_cell_kernel<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<N>::BYTES);
        if (e != cudaSuccess) return e;
        g_attr_done[dev] = 1;
    }
    const int64_t grid = (p.ntasks + C - 1) / C;
    if (p.ghosts) dg_cell_kernel<N, true><<<(unsigned)grid, THREADS, Smem<N>::BYTES, s>>>(p);
    else dg_cell_kernel<N, false><<<(unsigned)grid, THREADS, Smem<N>::BYTES, s>>>(p);
    return cudaGetLastError();
}

static int g_gen_attr_done[64];

// general-coefficient kernel (full / per-cell D; dg_gen.cuh)
cudaError_t DG_CAT(launch_gen_n, DG_N)(const KParams& p, cudaStream_t s)
{
    constexpr int N = DG_N;
    constexpr int C = GCfg<N>::C;
    if (p.ntasks <= 0) return cudaSuccess;
    if constexpr (N <= DG_REG_GMAX) {
        if (use_reg()) {
            const int64_t grid = (p.ntasks + REG_THREADS - 1) / REG_THREADS;
            if (p.ghosts) { cudaError_t e = reg_attr<N, true, true>(); if (e != cudaSuccess) return e; dg_reg_kernel<N, true, true><<<(unsigned)grid, REG_THREADS, RStage<N, true>::BYTES, s>>>(p); }
            else { cudaError_t e = reg_attr<N, true, false>(); if (e != cudaSuccess) return e; dg_reg_kernel<N, true, false><<<(unsigned)grid, REG_THREADS, RStage<N, true>::BYTES, s>>>(p); }
            return cudaGetLastError();
        }
    }
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !g_gen_attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(dg_gen_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             GSmem<N>::BYTES);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(dg_gen_kernel<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, GSmem<N>::BYTES);
        if (e != cudaSuccess) return e;
        g_gen_attr_done[dev] = 1;
    }
    const int64_t grid = (p.ntasks + C - 1) / C;
    if (p.ghosts) dg_gen_kernel<N, true><<<(unsigned)grid, C * GCfg<N>::TPC, GSmem<N>::BYTES, s>>>(p);
    else dg_gen_kernel<N, false><<<(unsigned)grid, C * GCfg<N>::TPC, GSmem<N>::BYTES, s>>>(p);
    return cudaGetLastError();
}

int DG_CAT(gen_info_n, DG_N)(LaunchInfo* info)
{
    constexpr int N = DG_N;
    if constexpr (N <= DG_REG_GMAX) if (use_reg()) {
        info->cells_per_cta = REG_THREADS;
        info->threads = REG_THREADS;
        info->smem = RStage<N, true>::BYTES;
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, dg_reg_kernel<N, true>) != cudaSuccess) return -3;
        info->regs = fa.numRegs;
        int blocks = 0;
        if (reg_attr<N, true, false>() != cudaSuccess) return -3;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, dg_reg_kernel<N, true>, REG_THREADS, RStage<N, true>::BYTES) !=
            cudaSuccess)
            return -3;
        info->ctas_per_sm = blocks;
        return 0;
    }
    info->cells_per_cta = GCfg<N>::C;
    info->threads = GCfg<N>::C * GCfg<N>::TPC;
    info->smem = GSmem<N>::BYTES;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, dg_gen_kernel<N, false>) != cudaSuccess) return -3;
    info->regs = fa.numRegs;
    if (cudaFuncSetAttribute(dg_gen_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GSmem<N>::BYTES) !=
        cudaSuccess)
        return -3;
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, dg_gen_kernel<N, false>, info->threads, GSmem<N>::BYTES) !=
        cudaSuccess)
        return -3;
    info->ctas_per_sm = blocks;
    return 0;
}

int DG_CAT(cell_info_n, DG_N)(LaunchInfo* info)
{
    constexpr int N = DG_N;
    if constexpr (N <= DG_REG_NMAX) if (use_reg()) {
        info->cells_per_cta = REG_THREADS;
        info->threads = REG_THREADS;
        info->smem = RStage<N, false>::BYTES;
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, dg_reg_kernel<N, false>) != cudaSuccess) return -3;
        info->regs = fa.numRegs;
        int blocks = 0;
        if (reg_attr<N, false, false>() != cudaSuccess) return -3;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, dg_reg_kernel<N, false>, REG_THREADS, RStage<N, false>::BYTES) != cudaSuccess)
            return -3;
        info->ctas_per_sm = blocks;
        return 0;
    }
#if DG_N == 8
    if (use_mma()) {
        constexpr int BYTES = m8::C * m8::PER_CELL * 8;
        info->cells_per_cta = m8::C;
        info->threads = 32 * m8::C;
        info->smem = BYTES;
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, m8::dg_cell_mma8) != cudaSuccess) return -3;
        info->regs = fa.numRegs;
        if (cudaFuncSetAttribute(m8::dg_cell_mma8, cudaFuncAttributeMaxDynamicSharedMemorySize, BYTES) != cudaSuccess)
            return -3;
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, m8::dg_cell_mma8, info->threads, BYTES) != cudaSuccess)
            return -3;
        info->ctas_per_sm = blocks;
        return 0;
    }
#endif
    info->cells_per_cta = Cfg<N>::C;
    info->threads = Cfg<N>::C * Cfg<N>::TPC;
    info->smem = Smem<N>::BYTES;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, dg_cell_kernel<N, false>) != cudaSuccess) return -3;
    info->regs = fa.numRegs;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !g_attr_done[dev]) {
        if (cudaFuncSetAttribute(dg_cell_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<N>::BYTES) !=
            cudaSuccess)
            return -3;
        g_attr_done[dev] = 1;
    }
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, dg_cell_kernel<N, false>, info->threads, Smem<N>::BYTES) !=
        cudaSuccess)
        return -3;
    info->ctas_per_sm = blocks;
    return 0;
}

}  // namespace dg
