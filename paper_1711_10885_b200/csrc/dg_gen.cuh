// General-coefficient cell kernel: y = A z for the WSIPG operator of arXiv 1711.10885 with
// a FULL symmetric diffusion tensor per cell (the paper's Problem A: "tensor-valued
// diffusion coefficients", "constant per cell", "weighted averaging across cell boundaries
// for discontinuous coefficients"), FP64, sm_100a.
//
// What changes against dg_cell_kernel (constant diagonal D):
//   * volume: the flux x^(r) = W (sum_s D_rs/(h_r h_s) d_s u - b_r/h_r u) couples the three
//     reference derivatives at every Gauss point (eq:gauss_points), so the
//     gradient is formed first (collocation derivatives Dc along x, y, z into three arrays),
//     the pointwise flux second and the transposed stages Dc_r^T last (eq:evalblf :425-444);
//   * faces: nu.D grad u = D_qq d_q u + D_qt1 d_t1 u + D_qt2 d_t2 u needs tangential
//     derivatives of both traces: on the neighbour side the face sum
//     factorization (normal first, :623-627) runs its tangential stages with V and G
//     (G_ij = theta'_j(xi_i)); on the own side Dc is applied along the face lines to the
//     extrapolated trace;
//   * weights w-+ = d+-/(d- + d+), penalty gamma = <d-, d+> sigma with d = nu^T D nu of each
//     side (reading C-5 for d- + d+ = 0);
//   * the test-gradient term -w J nu.D grad(phi) (eq:blf :312) lifts its normal part with
//     L'(s) along the normal and its tangential parts with Dc^T along the face lines, into
//     the quadrature-space accumulator before the V^T stages (normal direction LAST).
// Each cell still writes only its own y block once (owner computes, no atomics).
// Every array between stages is in sigma/delta form along each direction it has been evaluated
// in (dg_cell.cuh): the pointwise flux, the face fluxes and the lifts are linear with weights
// symmetric about the cell centre and the upwind / weight choices are per face, so they commute
// with the form; traces and lifts use rows built for it (Tab::Ls, Tab::Lsl).
#pragma once
#include "dg_cell.cuh"

namespace dg {

// index of D_rs in the 6-vector D00 D11 D22 D01 D02 D12
__host__ __device__ __forceinline__ constexpr int dsym(int r, int s)
{
    return r == s ? r : (r + s == 1 ? 3 : (r + s == 2 ? 4 : 5));
}

// t[i] = sum_j G_ij r[j] (G_{n-1-i,j} = (-1)^(j+1) G_ij: even-odd form)
template <int N>
__device__ __forceinline__ void g_fwd(const double (&Gh)[(N + 1) / 2][N], const double (&r)[N], double (&t)[N])
{
    constexpr int H = N / 2;
#pragma unroll
    for (int i = 0; i < H; ++i) {
        double E = 0.0, O = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (j & 1) O = fma(Gh[i][j], r[j], O);
            else E = fma(Gh[i][j], r[j], E);
        }
        t[i] = E + O;
        t[N - 1 - i] = O - E;
    }
    if (N & 1) {
        double O = 0.0;
#pragma unroll
        for (int j = 1; j < N; j += 2) O = fma(Gh[H][j], r[j], O);
        t[H] = O;
    }
}

// the same in sigma/delta form (position i < n/2: t_i + t_{n-1-i} = 2 O_i, position n-1-i:
// t_i - t_{n-1-i} = 2 E_i; Gs doubled, its middle row plain)
template <int N>
__device__ __forceinline__ void g_fwd_sd(const double (&Gs)[(N + 1) / 2][N], const double (&r)[N], double (&t)[N])
{
    constexpr int H = N / 2;
#pragma unroll
    for (int i = 0; i < H; ++i) {
        double E = 0.0, O = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (j & 1) O = fma(Gs[i][j], r[j], O);
            else E = fma(Gs[i][j], r[j], E);
        }
        t[i] = O;
        t[N - 1 - i] = E;
    }
    if (N & 1) {
        double O = 0.0;
#pragma unroll
        for (int j = 1; j < N; j += 2) O = fma(Gs[H][j], r[j], O);
        t[H] = O;
    }
}

// select among three / six register values by a runtime index (no local-memory array indexing)
__device__ __forceinline__ double sel3(double a0, double a1, double a2, int i) { return i == 0 ? a0 : (i == 1 ? a1 : a2); }
__device__ __forceinline__ int sel3i(int a0, int a1, int a2, int i) { return i == 0 ? a0 : (i == 1 ? a1 : a2); }
__device__ __forceinline__ double dsel(const double (&D)[6], int i)
{
    return i == 0 ? D[0] : i == 1 ? D[1] : i == 2 ? D[2] : i == 3 ? D[3] : i == 4 ? D[4] : D[5];
}

// pointer to the 6-vector D of the neighbour across face f (nullptr: no neighbour)
__device__ __forceinline__ const double* nb_dfield(const KParams& p, const int (&lc)[3], int64_t cell, int f,
                                                   unsigned nbmask)
{
    if (!((nbmask >> f) & 1u)) return nullptr;
    const int q = f >> 1, s = f & 1;
    const int nq = (int)sel3(p.nloc[0], p.nloc[1], p.nloc[2], q);
    const int lcq = sel3i(lc[0], lc[1], lc[2], q);
    const int64_t st = (q == 0) ? 1 : (q == 1) ? p.nloc[0] : p.nloc[0] * p.nloc[1];
    const int lq = lcq + (s ? 1 : -1);
    DG_ASSERT(lq >= -1 && lq <= nq);
    if (lq >= 0 && lq < nq) return p.Dfield + 6 * (cell + (s ? st : -st));
    if (p.wrap[q]) return p.Dfield + 6 * (cell + (s ? -(int64_t)(nq - 1) * st : (int64_t)(nq - 1) * st));
    const int64_t gi = (q == 0) ? (lc[1] + p.nloc[1] * lc[2]) : (q == 1) ? (lc[0] + p.nloc[0] * lc[2])
                                                                        : (lc[0] + p.nloc[0] * lc[1]);
    DG_ASSERT(p.Dghost[f] != nullptr);
    return p.Dghost[f] + 6 * gi;
}

// face-array layout of the general kernel: the fast kernel's, except n = 5, 6, 11 where the
// unpadded face arrays of FLay are slower here (different access mix: own traces, tangential
// derivatives; A-k4 31.7 -> 29.3, A-k5 28.5 -> 26.6, A-k10 29.1 -> 28.2 GDOF/s measured)
template <int N> struct GFLay : FLay<N> {};
template <int N> struct GFLayPad {
    static constexpr int RS = N + 1;
    static constexpr int ARR = N * RS + 1;
    static constexpr int SLOT = 12 * ARR;
    __device__ __forceinline__ static int at(int arr, int i1, int i2) { return arr * ARR + i1 + RS * i2; }
};
template <> struct GFLay<6> : GFLayPad<6> {};
// n = 7: i1 rotated by the face index (arr >> 1): the face passes' lines of consecutive faces
// land on different banks (bank-conflict model over those passes: 224 -> 134 wavefronts per
// cell; A-k6 27.8 -> 28.6 GDOF/s; the same idea measured slower at n = 5, 9 and neutral at 11,
// where the runtime mod costs more than the conflicts)
template <int N, int ARR, int CR> struct GFLayRot {
    static constexpr int SLOT = 12 * ARR;
    __device__ __forceinline__ static int at(int arr, int i1, int i2)
    {
        return arr * ARR + (i1 + CR * (arr >> 1)) % N + N * i2;
    }
};
template <> struct GFLay<7> : GFLayRot<7, 49, 6> {};
template <> struct GFLay<5> : GFLayPad<5> {};
// n = 8: a half-warp of the face passes (tk = lane: face f = tk / 8, line = tk % 8) covers the lines
// of two faces f, f + 1 (arrays 2f + c, 2f + 2 + c). Within an array the low three bits of the word
// index are i1 ^ i2 (a Latin square: a bijection along i1 and along i2) and bit 3 is i2 & 1, so one
// face's 8 lines along i1 or along i2, and 16 points (a, b) with b in {2h, 2h + 1}, take 8 (16)
// distinct banks; the array stride 68 = 4 mod 8 moves face f + 1 to the complementary 8 banks.
// Conflict free for every face-array access of this kernel (FLay<8> left 27 % of the shared-memory
// wavefronts as conflicts here, ncu A-k7), and cheaper index arithmetic than FLay<8>'s swizzle.
template <> struct GFLay<8> {
    static constexpr int ARR = 68;
    static constexpr int SLOT = 12 * ARR;
    __device__ __forceinline__ static int at(int arr, int i1, int i2) { return ARR * arr + 8 * i2 + (i1 ^ i2); }
};
template <> struct GFLay<11> : GFLayPad<11> {};
// n = 4: the face passes give one lane per line of faces f .. f + 3 on arrays 2f (+1): swizzle by
// the face index (arr >> 1) instead of the array index, so those 4 arrays take 4 different
// swizzles (with FLay<4>'s arr & 3, arrays 2f and 2f + 4 collided: ncu A-k3 24 % conflicts)
template <> struct GFLay<4> {
    static constexpr int SLOT = 12 * 16;
    __device__ __forceinline__ static int at(int arr, int i1, int i2)
    {
        const int s = (arr >> 1) & 3;
        return 16 * arr + (i1 ^ s) + 4 * (i2 ^ s);
    }
};

// launch configuration of the general kernel: the fast kernel's unless overridden per degree
#ifdef DG_GTPC
#define DG_GOVR(ov, d) (ov)
#else
#define DG_GOVR(ov, d) (d)
#endif
// (one pencil per thread is better than the fast kernel's 2 for n = 9, 10: A-k8 14.7 -> 31.4,
// A-k9 19.5 -> 27.5 GDOF/s;
// n = 6: 36 threads per cell (every thread a pencil), cells straddling warps: 2 cells per CTA A-k5
// 26.6 -> 28.5; 3 cells (108 threads) at 4 CTAs/SM 31.1 -> 34.3 (4 cells at 2 / 3 CTAs 29.0 / 32.6,
// 3 cells at 5 CTAs spills: 30.7); measured with tools/variant.py)
template <int N> struct GCfgD {
    static constexpr int TPC = (N == 6) ? 36 : (N == 9) ? 96 : (N == 10) ? 128 : Cfg<N>::TPC;
    static constexpr int P = (N == 6 || N == 9 || N == 10) ? 1 : Cfg<N>::P;
    static constexpr int C = (N == 6) ? 3 : (N == 9 || N == 10) ? 1 : Cfg<N>::C;
};
template <int N> struct GCfg {
    static constexpr int TPC = DG_GOVR(DG_GTPC, GCfgD<N>::TPC), P = DG_GOVR(DG_GP, GCfgD<N>::P),
                         C = DG_GOVR(DG_GC, GCfgD<N>::C);
};

// Per cell: three volume arrays (A0, X0, X1) and two face slots (NT, OT). d_z u is not stored:
// the pointwise step forms it on the thread's own z-pencil and applies the z role's Dc^T there
// (a fourth array cost 4 KB per cell at n = 8: 6 -> 8 CTAs per SM without it). n = 8 stages its
// TMA loads in OT (own block), X1 and A0 (x-neighbours), all free in phase 1, and its store in
// X0; only the mbarrier (16 B) is extra.
// How the face passes read this cell's tensor D (indexed by the face's direction, a run-time value):
// 0 from Dw (then in local memory), 1 a select chain over Dw in registers, 2 a shared-memory copy
// (A/B, tools/variant.py -DDG_DW_SEL: A-k3 36.8 -> 38.0 (2); A-k4 33.1 -> 34.4 (1), 34.2 (2);
// A-k6 30.7 -> 31.3 (1), 31.6 (2); A-k7 50.0 -> 45.0 (1), 45.9 (2), A-k8 35.3 -> 33.9 (2), A-k5 34.2 -> 30.8 (1),
// A-k9 35.2 -> 33.4 (1), A-k10 36.5 -> 33.4 (1), 34.9 (2): spills / registers)
#ifndef DG_DW_SEL
#define DG_DW_SEL ((DG_N) == 5 ? 1 : ((DG_N) == 4 || (DG_N) == 7) ? 2 : 0)
#endif
template <int N>
struct GSmem {
    static constexpr int PER_CELL = 3 * Lay<N>::SLOT + 2 * GFLay<N>::SLOT;
    static constexpr int STAGE = (N >= 7) ? 2 : 0;   // the mbarrier (n = 8: TMA; n = 7, 9, 11: bulk copies)
    static constexpr int BYTES = GCfg<N>::C * PER_CELL * 8 + STAGE * 8 + (DG_DW_SEL == 2 ? GCfg<N>::C * 64 : 0);
};

template <int N, bool GH>
#ifndef DG_GMB
#define DG_GMB ((DG_N) == 4 ? 12 : (DG_N) == 6 ? 4 : (DG_N) == 8 ? 8 : (DG_N) == 10 ? 5 : (DG_N) == 11 ? 3 : 1)   // min CTAs per SM (n = 4: A-k3 30.5 -> 31.0; n = 8: the 8 CTAs its shared memory allows; n = 10: A-k9 29.7 -> 31.0; n = 11: the 3 its shared memory allows, A-k10 35.4 -> 36.1)
#endif
__global__ void __launch_bounds__(GCfg<N>::C * GCfg<N>::TPC, DG_GMB)
dg_gen_kernel(const __grid_constant__ KParams p)
{
    constexpr int TPC = GCfg<N>::TPC, P = GCfg<N>::P, C = GCfg<N>::C;
    constexpr int NN = N * N;
    static_assert(TPC * P >= NN, "pencil slots");
    extern __shared__ double smem[];
    const Tab<N>& T = g_tab;

    const int tid = threadIdx.x;
    const int slot = tid / TPC;
    const int lane = tid - slot * TPC;
    double* A0 = smem + slot * GSmem<N>::PER_CELL;   // u, then the quadrature-space accumulator
    double* X0 = A0 + Lay<N>::SLOT;                  // d_x u -> x^(1)   (also a stage temporary)
    double* X1 = X0 + Lay<N>::SLOT;                  // d_y u -> x^(2)
    double* NT = X1 + Lay<N>::SLOT;                  // neighbour face arrays (2 per face)
    double* OT = NT + GFLay<N>::SLOT;                 // own face arrays (2 per face)
    auto csync = [&]() {
        if (32 % TPC == 0) __syncwarp(); else __syncthreads();   // a cell within one warp, else CTA-wide
    };

    unsigned task = blockIdx.x * (unsigned)C + (unsigned)slot;
    const bool valid = task < (unsigned)p.ntasks;
    if (!valid) task = (unsigned)p.ntasks - 1u;
    int lc[3];
    {
        const unsigned e = p.task_list ? (unsigned)p.task_list[task] : 0u;
        if (p.task_list) {
            const unsigned nx = (unsigned)p.nloc[0], ny = (unsigned)p.nloc[1];
            lc[0] = (int)(e % nx);
            lc[1] = (int)((e / nx) % ny);
            lc[2] = (int)(e / (nx * ny));
        } else {
            decode_task(p, task, lc);
        }
    }
    const int64_t n3 = (int64_t)NN * N;
    const int64_t cell = lc[0] + p.nloc[0] * (lc[1] + p.nloc[1] * (int64_t)lc[2]);
    DG_ASSERT(lc[0] >= 0 && lc[0] < p.nloc[0] && lc[1] >= 0 && lc[1] < p.nloc[1] && lc[2] >= 0 && lc[2] < p.nloc[2]);
    const double* zc = p.z + cell * n3;
    const bool do_int = (p.mask & 2u) != 0, do_bnd = (p.mask & 4u) != 0, do_vol = (p.mask & 1u) != 0;

    unsigned nbmask = 0;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        const int q = f >> 1, s = f & 1;
        const int64_t g = p.gofs[q] + lc[q] + (s ? 1 : -1);
        if (p.per[q] || (g >= 0 && g < p.gcells[q])) nbmask |= 1u << f;
    }
    const unsigned nbi = do_int ? nbmask : 0u;                   // neighbour traces needed
    const unsigned fact = (do_int ? nbmask : 0u) | (do_bnd ? (~nbmask & 63u) : 0u);   // faces with a term
    double Dw[6];                                                // this cell's tensor
#pragma unroll
    for (int i = 0; i < 6; ++i) Dw[i] = __ldg(p.Dfield + 6 * cell + i);
#if DG_DW_SEL == 1
    // face passes index the tensor by the face's direction: a select chain keeps Dw in registers
    // (a dynamic index would place it in local memory)
    auto dwv = [&](int i) {
        double r = Dw[0];
#pragma unroll
        for (int j = 1; j < 6; ++j) r = (i == j) ? Dw[j] : r;
        return r;
    };
#elif DG_DW_SEL == 2
    // face passes index the tensor by the face's direction: read it from a shared copy (a dynamic
    // index into Dw would place Dw in local memory); first read after the phase barriers
    double* Dsm = smem + C * GSmem<N>::PER_CELL + GSmem<N>::STAGE + 8 * slot;
    if (lane < 6) Dsm[lane] = __ldg(p.Dfield + 6 * cell + lane);
    auto dwv = [&](int i) { return Dsm[i]; };
#else
    auto dwv = [&](int i) { return Dw[i]; };
#endif
    // The face passes give work item tk = lane (one pass over 6 n face lines when TPC >= 6 n) the
    // lines of face f = lane / n: that face's neighbour tensor is loaded here, long before its use
    // (the dependent L2 loads in the passes were long-scoreboard stalls)
    constexpr bool PREF = TPC >= 6 * N && N != 10;   // (n = 10: A-k9 -3.6 %; A-k7 +6.4 %, A-k5 +3.5 %)
    double pf_qq = 0.0, pf_q1 = 0.0, pf_q2 = 0.0;
    if (PREF && lane < 6 * N) {
        const int f = lane / N, q = f >> 1;
        const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
        if ((nbmask >> f) & 1u) {
            const double* Dn = nb_dfield(p, lc, cell, f, nbmask);
            pf_qq = __ldg(Dn + q);
            pf_q1 = __ldg(Dn + dsym(q, t1));
            pf_q2 = __ldg(Dn + dsym(q, t2));
        }
    }

    int pa[P], pb[P];
    bool act[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const int pc = lane + k * TPC;
        act[k] = pc < NN;
        const int pcc = act[k] ? pc : 0;
        pa[k] = pcc % N;
        pb[k] = pcc / N;
    }

    double r[P][N], t[P][N];
    // TMA staging (n = 8): own block (STG = OT) and the local x-neighbours' blocks (X1, A0), all
    // free in P1; the mbarrier after the cell's arrays
    double* STG = nullptr;
    double* XH = A0;
    bool tma_x = false;
    if constexpr (N == 8 && C == 1) {
        if (p.tma) {
            STG = OT;
            tma_x = tma::stage_x(p, STG, X1, XH, tid, lc, cell, nbi,
                                 reinterpret_cast<uint64_t*>(smem + GSmem<N>::PER_CELL));
        }
    }
    // n = 7, 9, 11: the own block by one bulk copy into a linear image in OT (free in P1), y out of
    // X0 by one bulk copy (dg_cell.cuh, namespace bulk): A-k6 / k8 / k10 29.8 -> 30.7, 33.5 -> 35.0,
    // 30.6 -> 34.1 GDOF/s; n = 10 measured 34.9 -> 33.7: off
    constexpr bool BULK = (N == 7 || N == 9 || N == 11) && C == 1;
    static_assert(!BULK || (GFLay<N>::SLOT >= NN * N + 1 && Lay<N>::SLOT >= NN * N + 1), "block images");
    double* SB = nullptr;
    double *SL = nullptr, *SH = nullptr;   // the local x-neighbours' images (X1, A0: free in P1)
    bulk::Span bs{}, bl{}, bh{};
    bool bulk_x = false;
    if constexpr (BULK) {
        if (p.tma) {
            uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + GSmem<N>::PER_CELL);
            const int nq = (int)p.nloc[0];
            const bool hl = (nbi & 1u) != 0, hh = (nbi & 2u) != 0;
            const bool ll = hl && (lc[0] > 0 || p.wrap[0]), lh = hh && (lc[0] + 1 < nq || p.wrap[0]);
            // x-neighbours staged too (n = 11 only: A-k10 34.1 -> 35.6 GDOF/s; n = 7, 9 -0.5 / -0.9 %)
            // when every x-neighbour is on this rank (ghosts: per-thread loads)
            bulk_x = N == 11 && (ll || !hl) && (lh || !hh);
            const double* zlo = p.z + ((lc[0] > 0) ? cell - 1 : cell + (nq - 1)) * n3;
            const double* zhi = p.z + ((lc[0] + 1 < nq) ? cell + 1 : cell - (nq - 1)) * n3;
            bs = bulk::span<N>(zc, OT);
            SB = OT + bs.sh;
            if (bulk_x) {
                bl = bulk::span<N>(zlo, X1);
                bh = bulk::span<N>(zhi, A0);
                SL = X1 + bl.sh;
                SH = A0 + bh.sh;
            }
            if (tid == 0) tma::mbar_init_n(mbar, 1);
            __syncthreads();
            if (tid == 0) {
                const bool xl = bulk_x && hl, xh = bulk_x && hh;
                tma::expect_tx(mbar, bs.bytes + (xl ? bl.bytes : 0u) + (xh ? bh.bytes : 0u));
                bulk::load(SB + bs.hd, zc + bs.hd, bs.bytes, mbar);
                if (xl) bulk::load(SL + bl.hd, zlo + bl.hd, bl.bytes, mbar);
                if (xh) bulk::load(SH + bh.hd, zhi + bh.hd, bh.bytes, mbar);
            }
            tma::wait(mbar, 0);
            if (bulk_x) {   // the plain leading / trailing doubles of the neighbour images
                if (bl.hd && tid == 0) SL[0] = __ldg(zlo);
                if (bh.hd && tid == 0) SH[0] = __ldg(zhi);
                if (bl.tl && tid == 0) SL[n3 - 1] = __ldg(zlo + n3 - 1);
                if (bh.tl && tid == 0) SH[n3 - 1] = __ldg(zhi + n3 - 1);
                if ((bl.hd | bh.hd | bl.tl | bh.tl) && hl | hh) __syncthreads();
            }
        }
    }
    // ---------------------------------------------------------------- P1-P3: u at the Gauss points
    {
        double rl[P][N], rh[P][N];
        unsigned gm = 0;   // ghost neighbours (traces from the halo; x-ghosts are never TMA-staged)
        if (tma_x) {
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const int L = pa[k] + N * pb[k];
#pragma unroll
                for (int e = 0; e < N; e += 2) {
                    const double2 a = tma::line2(STG, L, e), lo = tma::line2(X1, L, e), hi = tma::line2(XH, L, e);
                    r[k][e] = a.x; r[k][e + 1] = a.y;
                    rl[k][e] = lo.x; rl[k][e + 1] = lo.y;
                    rh[k][e] = hi.x; rh[k][e + 1] = hi.y;
                }
            }
        } else {
            if (bulk_x) {
#pragma unroll
                for (int k = 0; k < P; ++k) {
                    const int o = N * (pa[k] + N * pb[k]);
                    if (N % 2 == 0) {
#pragma unroll
                        for (int e = 0; e < N; e += 2) {
                            const double2 lo = *reinterpret_cast<const double2*>(SL + o + e);
                            const double2 hi = *reinterpret_cast<const double2*>(SH + o + e);
                            rl[k][e] = lo.x; rl[k][e + 1] = lo.y;
                            rh[k][e] = hi.x; rh[k][e + 1] = hi.y;
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < N; ++e) {
                            rl[k][e] = SL[o + e];
                            rh[k][e] = SH[o + e];
                        }
                    }
                }
            } else {
                gm = nb_load<N, P, GH>(p, zc, n3, 0, lc, nbi, pa, pb, act, rl, rh);
            }
#pragma unroll
            for (int k = 0; k < P; ++k) {
                if (STG) {
                    const int L = pa[k] + N * pb[k];
#pragma unroll
                    for (int e = 0; e < N; e += 2) {
                        const double2 a = tma::line2(STG, L, e);
                        r[k][e] = a.x; r[k][e + 1] = a.y;
                    }
                    continue;
                }
                if (BULK && SB) {
                    const double* src = SB + N * (pa[k] + N * pb[k]);
                    if (N % 2 == 0) {
#pragma unroll
                        for (int e = 0; e < N; e += 2) {
                            const double2 v = act[k] ? *reinterpret_cast<const double2*>(src + e) : make_double2(0.0, 0.0);
                            r[k][e] = v.x;
                            r[k][e + 1] = v.y;
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? src[e] : 0.0;
                    }
                    continue;
                }
                const double* src = zc + N * (pa[k] + N * pb[k]);
#pragma unroll
                for (int e = 0; e < N; ++e) r[k][e] = act[k] ? __ldg(src + e) : 0.0;
            }
            if (BULK && SB) {   // the plain leading / trailing doubles of the block
                if (bs.hd && lane == 0) r[0][0] = __ldg(zc);
                if (bs.tl && lane == (NN - 1) % TPC) r[(NN - 1) / TPC][N - 1] = __ldg(zc + NN * N - 1);
            }
        }
        v_fwd_sd<N, P>(T.Vs[0], r, t);
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (act[k])
#pragma unroll
                for (int e = 0; e < N; ++e) X0[Lay<N>::at(e, pa[k], pb[k])] = t[k][e];
        nb_contract<N, P, GFLay<N>>(T, NT, 0, nbi, pa, pb, act, rl, rh, gm);
        if (DG_EARLYNB) gm = nb_load<N, P, GH>(p, zc, n3, 1, lc, nbi, pa, pb, act, rl, rh);
        csync();

        if (!DG_EARLYNB) gm = nb_load<N, P, GH>(p, zc, n3, 1, lc, nbi, pa, pb, act, rl, rh);
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int e = 0; e < N; ++e) r[k][e] = act[k] ? X0[Lay<N>::at(pa[k], e, pb[k])] : 0.0;
        v_fwd_sd<N, P>(T.Vs[1], r, t);
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (act[k])
#pragma unroll
                for (int e = 0; e < N; ++e) X1[Lay<N>::at(pa[k], e, pb[k])] = t[k][e];
        nb_contract<N, P, GFLay<N>>(T, NT, 1, nbi, pa, pb, act, rl, rh, gm);
        if (DG_EARLYNB) gm = nb_load<N, P, GH>(p, zc, n3, 2, lc, nbi, pa, pb, act, rl, rh);
        csync();

        if (!DG_EARLYNB) gm = nb_load<N, P, GH>(p, zc, n3, 2, lc, nbi, pa, pb, act, rl, rh);
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int e = 0; e < N; ++e) r[k][e] = act[k] ? X1[Lay<N>::at(pa[k], pb[k], e)] : 0.0;
        nb_contract<N, P, GFLay<N>>(T, NT, 2, nbi, pa, pb, act, rl, rh, gm);
    }
    v_fwd_sd<N, P>(T.Vs[2], r, t);                               // t = u on this thread's z-pencils
    {
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (act[k]) {
#pragma unroll
                for (int e = 0; e < N; ++e) A0[Lay<N>::at(pa[k], pb[k], e)] = t[k][e];
                // own z-face traces: u and the reference normal derivative at z = 0, 1
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    OT[GFLay<N>::at(2 * (4 + s), pa[k], pb[k])] = dot<N>(T.Ls[0][s], t[k]);
                    OT[GFLay<N>::at(2 * (4 + s) + 1, pa[k], pb[k])] = dot<N>(T.Ls[0][2 + s], t[k]);
                }
            }
    }
    csync();

    // ---------------------------------------------------------------- P4: d_x u, d_y u, own x/y traces;
    //                                                                  neighbour tangential stage 1
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int e = 0; e < N; ++e)
                r[k][e] = act[k] ? A0[q == 0 ? Lay<N>::at(e, pa[k], pb[k]) : Lay<N>::at(pa[k], e, pb[k])] : 0.0;
        {
            double z0[P][(N / 2) > 0 ? N / 2 : 1], zm[P];
            c_apply_s<N, P, false>(T.Dcs[1 + q], r, t, z0, z0, zm);
        }
        double* X = q == 0 ? X0 : X1;
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (act[k]) {
#pragma unroll
                for (int e = 0; e < N; ++e)
                    X[q == 0 ? Lay<N>::at(e, pa[k], pb[k]) : Lay<N>::at(pa[k], e, pb[k])] = t[k][e];
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    OT[GFLay<N>::at(2 * (2 * q + s), pa[k], pb[k])] = dot<N>(T.Ls[1][s], r[k]);
                    OT[GFLay<N>::at(2 * (2 * q + s) + 1, pa[k], pb[k])] = dot<N>(T.Ls[1][2 + s], r[k]);
                }
            }
    }
    // neighbour stage 1 (lines along i1): Va = V a, E = D+_qq/h_q V d + D+_qt1/h_t1 G a
    for (int tk = lane; tk < 6 * N; tk += TPC) {
        const int f = tk / N, line = tk - f * N, q = f >> 1;
        if (!((nbi >> f) & 1u)) continue;
        const int t1 = (q == 0) ? 1 : 0;
        double cqq, cq1;
        if (PREF) {
            cqq = pf_qq * p.hinv[q];
            cq1 = pf_q1 * p.hinv[t1];
        } else {
            const double* Dn = nb_dfield(p, lc, cell, f, nbmask);
            cqq = __ldg(Dn + q) * p.hinv[q];
            cq1 = __ldg(Dn + dsym(q, t1)) * p.hinv[t1];
        }
        double rr[1][N], tt[1][N], ga[N];
#pragma unroll
        for (int e = 0; e < N; ++e) rr[0][e] = NT[GFLay<N>::at(2 * f, e, line)];
        g_fwd_sd<N>(T.Gs, rr[0], ga);
        v_fwd_sd<N, 1>(T.Vs[3], rr, tt);
#pragma unroll
        for (int e = 0; e < N; ++e) {
            NT[GFLay<N>::at(2 * f, e, line)] = tt[0][e];
            rr[0][e] = NT[GFLay<N>::at(2 * f + 1, e, line)];
        }
        v_fwd_sd<N, 1>(T.Vs[4], rr, tt);
#pragma unroll
        for (int e = 0; e < N; ++e) NT[GFLay<N>::at(2 * f + 1, e, line)] = fma(cqq, tt[0][e], cq1 * ga[e]);
    }
    csync();

    // ---------------------------------------------------------------- P5: neighbour stage 2, own pass A,
    //                                                                  pointwise volume data
    for (int tk = lane; tk < 12 * N; tk += TPC) {
        const int f = (tk >= 6 * N) ? (tk - 6 * N) / N : tk / N;
        const int line = tk % N, q = f >> 1;
        const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
        if (tk < 6 * N) {
            // neighbour stage 2 (lines along i2): u+ = V Va, s+ = V E + D+_qt2/h_t2 G Va
            if (!((nbi >> f) & 1u)) continue;
            const double cq2 = (PREF ? pf_q2 : __ldg(nb_dfield(p, lc, cell, f, nbmask) + dsym(q, t2))) * p.hinv[t2];
            double rr[1][N], tt[1][N], va[N], gv[N];
#pragma unroll
            for (int e = 0; e < N; ++e) va[e] = NT[GFLay<N>::at(2 * f, line, e)];
#pragma unroll
            for (int e = 0; e < N; ++e) rr[0][e] = va[e];
            v_fwd_sd<N, 1>(T.Vs[5], rr, tt);
#pragma unroll
            for (int e = 0; e < N; ++e) {
                NT[GFLay<N>::at(2 * f, line, e)] = tt[0][e];
                rr[0][e] = NT[GFLay<N>::at(2 * f + 1, line, e)];
            }
            v_fwd_sd<N, 1>(T.Vs[6], rr, tt);
            g_fwd_sd<N>(T.Gs, va, gv);
#pragma unroll
            for (int e = 0; e < N; ++e) NT[GFLay<N>::at(2 * f + 1, line, e)] = fma(cq2, gv[e], tt[0][e]);
        } else {
            // own pass A (lines along i1): s_part = D_qq/h_q d_n u + D_qt1/h_t1 Dc u-
            if (!((fact >> f) & 1u)) continue;
            const double cqq = dwv(q) * p.hinv[q], cq1 = dwv(dsym(q, t1)) * p.hinv[t1];
            double rr[1][N], tt[1][N];
#pragma unroll
            for (int e = 0; e < N; ++e) rr[0][e] = OT[GFLay<N>::at(2 * f, e, line)];
            double z0[1][(N / 2) > 0 ? N / 2 : 1], zm[1];
            c_apply_s<N, 1, false>(T.Dcs[3], rr, tt, z0, z0, zm);
#pragma unroll
            for (int e = 0; e < N; ++e) {
                const int ix = GFLay<N>::at(2 * f + 1, e, line);
                OT[ix] = fma(cqq, OT[ix], cq1 * tt[0][e]);
            }
        }
    }
    {
        // x^(r) = W (sum_s D_rs/(h_r h_s) d_s u - b_r/h_r u)   (eq:gauss_points) on the thread's
        // z-pencils; d_z u = Dc u along the pencil here; the z role's Dc^T x^(3) is applied in
        // registers and A0 = W c u + Dc_z^T x^(3) (the x, y roles and the z lifts add later)
        double Dh[3][3];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr)
#pragma unroll
            for (int ss = 0; ss < 3; ++ss) Dh[rr][ss] = dwv(dsym(rr, ss)) * (p.hinv[rr] * p.hinv[ss]);
        double u[P][N], g[P][N];
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int e = 0; e < N; ++e) u[k][e] = act[k] ? A0[Lay<N>::at(pa[k], pb[k], e)] : 0.0;
        {
            double z0[P][(N / 2) > 0 ? N / 2 : 1], zm[P];
            c_apply_s<N, P, false>(T.Dcs[0], u, g, z0, z0, zm);   // d_z u
        }
        double cu[P][(N / 2) > 0 ? N / 2 : 1], cl[P][(N / 2) > 0 ? N / 2 : 1], cm[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const double wab = do_vol ? p.dT * T.w[pa[k]] * T.w[pb[k]] : 0.0;
#pragma unroll
            for (int e = 0; e < N; ++e) {
                const int ix = Lay<N>::at(pa[k], pb[k], e);
                const double W = wab * T.w[e];
                const double uu = u[k][e], g0 = act[k] ? X0[ix] : 0.0, g1 = act[k] ? X1[ix] : 0.0, g2 = g[k][e];
                if (act[k]) {
                    X0[ix] = W * (Dh[0][0] * g0 + Dh[0][1] * g1 + Dh[0][2] * g2 - p.kb[0] * uu);
                    X1[ix] = W * (Dh[1][0] * g0 + Dh[1][1] * g1 + Dh[1][2] * g2 - p.kb[1] * uu);
                }
                g[k][e] = W * (Dh[2][0] * g0 + Dh[2][1] * g1 + Dh[2][2] * g2 - p.kb[2] * uu);   // x^(3)
                const double wcu = W * p.c * uu;
                if (e < N / 2) cu[k][e] = wcu;                  // added to output e (< n/2)
                else if (2 * e + 1 == N) cm[k] = wcu;           // the middle (odd n)
                else cl[k][N - 1 - e] = wcu;                    // output e = n-1-i
            }
        }
        c_apply_s<N, P, true>(T.DcTs[4], g, u, cu, cl, cm);      // u <- W c u + Dc_z^T x^(3)
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (act[k])
#pragma unroll
                for (int e = 0; e < N; ++e) A0[Lay<N>::at(pa[k], pb[k], e)] = u[k][e];
    }
    csync();

    // ---------------------------------------------------------------- P6: own pass B, fluxes, Dc^T along i2
    for (int tk = lane; tk < 6 * N; tk += TPC) {
        const int f = tk / N, line = tk - f * N, q = f >> 1, sd = f & 1;
        if (!((fact >> f) & 1u)) continue;
        const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
        const bool interior = (nbmask >> f) & 1u;
        const double dme = dwv(q);
        const double cq2 = dwv(dsym(q, t2)) * p.hinv[t2];
        const double cn = dme * p.hinv[q], c1 = dwv(dsym(q, t1)) * p.hinv[t1];
        double uo[N], so[N], cv[N];
        {
            double rr[1][N], tt[1][N];
#pragma unroll
            for (int e = 0; e < N; ++e) uo[e] = rr[0][e] = OT[GFLay<N>::at(2 * f, line, e)];
            double z0[1][(N / 2) > 0 ? N / 2 : 1], zm[1];
            c_apply_s<N, 1, false>(T.Dcs[4], rr, tt, z0, z0, zm);
#pragma unroll
            for (int e = 0; e < N; ++e) so[e] = fma(cq2, tt[0][e], OT[GFLay<N>::at(2 * f + 1, line, e)]);
        }
        double dnb = 0.0;
        if (interior) dnb = PREF ? pf_qq : __ldg(nb_dfield(p, lc, cell, f, nbmask) + q);
        const double dm = sd ? dme : dnb, dp = sd ? dnb : dme;     // delta of T-, T+
        const double dsum = dm + dp;
        const double rsum = dsum == 0.0 ? 0.0 : 1.0 / dsum;
        const double wm = dsum == 0.0 ? 0.5 : dp * rsum, wp = dsum == 0.0 ? 0.5 : dm * rsum;   // C-5
        const double gam = (interior ? 2.0 * dm * dp * rsum : dme) * p.sigq[q];
        const double bq = p.bq[q];
        // The face terms as one branch-free expression in the own (o) and neighbour (n) traces,
        // with per-line scalars (sg = +-1: the own side is T- for sd = 1):
        //   interior: J = u- - u+ = sg (uo - un), {nu.D grad u}_w = ws so + wn sn,
        //             upwind Phi = bq u_up, cv = sg Wf (Phi - {.}_w + gam J),
        //             coef = -Wf w_self J;
        //   boundary (weak Dirichlet, outward normal sg): cv = Wf (Phi - sg so + gam uo) with
        //             Phi = max(sg bq, 0) uo, coef = -Wf sg uo  (un = sn = 0, ws = 1, wn = 0).
        const double sg = sd ? 1.0 : -1.0;
        const bool own_up = interior ? ((bq >= 0.0) == (sd != 0)) : (sg * bq >= 0.0);
        const double ws = interior ? (sd ? wm : wp) : 1.0, wn = interior ? (sd ? wp : wm) : 0.0;
        // com = cv / (sg Wf) = ko uo + kn un - (ws so + wn sn)   (sg^2 = 1 folds the boundary case)
        const double ko = (own_up ? bq : 0.0) + sg * gam;
        const double kn = interior ? ((own_up ? 0.0 : bq) - sg * gam) : 0.0;
        const double cw = ws;                                // coef = -Wf sg cw (uo - un)
        const double Wl = p.dF[q] * T.w[line] * sg;
        double c2[N];
#pragma unroll
        for (int e = 0; e < N; ++e) {
            const double Wf = Wl * T.w[e];                         // face point (i1 = line, i2 = e), times sg
            const double un = interior ? NT[GFLay<N>::at(2 * f, line, e)] : 0.0;
            const double sn = interior ? NT[GFLay<N>::at(2 * f + 1, line, e)] : 0.0;
            const double com = fma(ko, uo[e], fma(kn, un, -fma(ws, so[e], wn * sn)));
            cv[e] = Wf * com;
            const double coef = -Wf * cw * (uo[e] - un);       // coefficient of e_q.D grad(phi)
            OT[GFLay<N>::at(2 * f + 1, line, e)] = coef * cn;         // normal part (lifted with L')
            NT[GFLay<N>::at(2 * f, line, e)] = coef * c1;             // t1 part (Dc^T along i1 in P7)
            c2[e] = coef * cq2;                                      // t2 part (Dc^T along i2 below)
        }
        {
            double rr[1][N], tt[1][N];
#pragma unroll
            for (int e = 0; e < N; ++e) rr[0][e] = c2[e];
            double z0[1][(N / 2) > 0 ? N / 2 : 1], zm[1];
            c_apply_s<N, 1, false>(T.DcTs[0], rr, tt, z0, z0, zm);   // tangential test derivative along i2
#pragma unroll
            for (int e = 0; e < N; ++e) OT[GFLay<N>::at(2 * f, line, e)] = cv[e] + tt[0][e];
        }
    }
    csync();

    // ---------------------------------------------------------------- P7: Dc^T along i1 of the t1 parts
    for (int tk = lane; tk < 6 * N; tk += TPC) {
        const int f = tk / N, line = tk - f * N;
        if (!((fact >> f) & 1u)) continue;
        double rr[1][N], tt[1][N];
#pragma unroll
        for (int e = 0; e < N; ++e) rr[0][e] = NT[GFLay<N>::at(2 * f, e, line)];
        double z0[1][(N / 2) > 0 ? N / 2 : 1], zm[1];
        c_apply_s<N, 1, false>(T.DcTs[1], rr, tt, z0, z0, zm);
#pragma unroll
        for (int e = 0; e < N; ++e) OT[GFLay<N>::at(2 * f, e, line)] += tt[0][e];
    }
    csync();

    // ---------------------------------------------------------------- P8-P10: roles, A0 += Dc_q^T x^(q) + lifts
    // (the z role's Dc^T x^(3) is already in A0: that role adds the z-face lifts only)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        double* X = q == 0 ? X0 : X1;
        auto at = [&](int k, int e) {
            return q == 0 ? Lay<N>::at(e, pa[k], pb[k]) : (q == 1 ? Lay<N>::at(pa[k], e, pb[k]) : Lay<N>::at(pa[k], pb[k], e));
        };
        if (q < 2) {
#pragma unroll
            for (int k = 0; k < P; ++k)
#pragma unroll
                for (int e = 0; e < N; ++e) r[k][e] = act[k] ? X[at(k, e)] : 0.0;
            double z0[P][(N / 2) > 0 ? N / 2 : 1], zm[P];
            c_apply_s<N, P, false>(T.DcTs[2 + q], r, t, z0, z0, zm);
        } else {
#pragma unroll
            for (int k = 0; k < P; ++k)
#pragma unroll
                for (int e = 0; e < N; ++e) t[k][e] = act[k] ? A0[at(k, e)] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < P; ++k) {
            if (!act[k]) continue;
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int f = 2 * q + s;
                if (!((fact >> f) & 1u)) continue;
                const double cv = OT[GFLay<N>::at(2 * f, pa[k], pb[k])];
                const double cg = OT[GFLay<N>::at(2 * f + 1, pa[k], pb[k])];
#pragma unroll
                for (int e = 0; e < N; ++e) t[k][e] = fma(cv, T.Lsl[s][e], fma(cg, T.Lsl[2 + s][e], t[k][e]));
            }
        }
        if (q < 2) {
#pragma unroll
            for (int k = 0; k < P; ++k)
                if (act[k])
#pragma unroll
                    for (int e = 0; e < N; ++e) A0[at(k, e)] += t[k][e];
            csync();
        }
    }
    // ---------------------------------------------------------------- P10-P12: V^T along z, y, x; store
    v_bwd_sd<N, P>(T.Vh[9], t, r);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A0[Lay<N>::at(pa[k], pb[k], e)] = r[k][e];
    csync();
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(pa[k], e, pb[k])] : 0.0;
    v_bwd_sd<N, P>(T.Vh[10], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A0[Lay<N>::at(pa[k], e, pb[k])] = t[k][e];
    csync();
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(e, pa[k], pb[k])] : 0.0;
    v_bwd_sd<N, P>(T.Vh[11], r, t);
    if constexpr (N == 8 && C == 1) {
        if (STG && p.tma == 2 && p.epi == 0) {   // y through a staging block (X0, free) and one TMA store
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const int L = pa[k] + N * pb[k];
#pragma unroll
                for (int e = 0; e < N; e += 2) tma::put2(X0, L, e, t[k][e], t[k][e + 1]);
            }
            tma::store_block(p, X0, tid, cell);
            return;
        }
    }
    if constexpr (BULK) {
        if (p.tma == 2 && p.epi == 0) {   // y through a linear image in X0 (free) and one bulk store
            double* yc = p.y + cell * n3;
            const bulk::Span ys = bulk::span<N>(yc, X0);
            double* S = X0 + ys.sh;
#pragma unroll
            for (int k = 0; k < P; ++k) {
                if (!act[k]) continue;
                double* dst = S + N * (pa[k] + N * pb[k]);
                if (N % 2 == 0) {
#pragma unroll
                    for (int e = 0; e < N; e += 2) *reinterpret_cast<double2*>(dst + e) = make_double2(t[k][e], t[k][e + 1]);
                } else {
#pragma unroll
                    for (int e = 0; e < N; ++e) dst[e] = t[k][e];
                }
            }
            if (valid) {
                if (ys.hd && lane == 0) __stcs(yc, t[0][0]);
                if (ys.tl && lane == (NN - 1) % TPC) __stcs(yc + NN * N - 1, t[(NN - 1) / TPC][N - 1]);
            }
            tma::fence_async();
            __syncthreads();
            if (valid && tid == 0) bulk::store(yc + ys.hd, S + ys.hd, ys.bytes);
            return;
        }
    }
    if (valid) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
            if (!act[k]) continue;
            const int64_t off = cell * n3 + N * (pa[k] + N * pb[k]);
            double* yc = p.y + off;
            epilogue<N>(p, off, t[k]);
#pragma unroll
            for (int e = 0; e < N; ++e) __stcs(yc + e, t[k][e]);
        }
    }
}

}  // namespace dg
