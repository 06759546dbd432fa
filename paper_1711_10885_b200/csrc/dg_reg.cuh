// Register-resident cell kernel for the smallest bases: one THREAD per cell (constant diagonal D,
// the fast path of dg_cell.cuh, for n <= DG_REG_NMAX; GEN = true: full / per-cell tensors, the
// general path of dg_gen.cuh, for n <= DG_REG_GMAX), the whole n^3 block and every
// intermediate array in registers, no shared memory and no barriers.
//
// Why: at n = 2 a pencil is 2 points, so the pencil kernel spends most of its issue slots on
// shared-memory traffic, addresses and barriers (ncu, C4 k = 1: issue 83 %, FP64 pipe 40 %,
// smem wavefronts 77 %). Here the same arithmetic runs per cell with the 1D matrices reused
// across all n^2 lines of a stage.
//
// Same method and same readings as dg_cell_kernel:
//   u = (V x V x V) z at the Gauss points; d_q u = Dc along q (collocation derivative);
//   x^(q) = W (D_qq/h_q^2 d_q u - b_q/h_q u)  (eq:gauss_points);
//   own traces u(s), d_q u(s) by Lagrange extrapolation of the Gauss-point values along the
//   normal; neighbour traces by the face sum factorization with the normal FIRST
//   (theta(1-s), theta'(1-s) on the neighbour's normal index, then V along both tangentials,
//   PAPER.md:623-627); SIPG + upwind flux (flux_interior / flux_boundary, eq:blf :301-315);
//   lift of the face coefficients into the quadrature-space accumulator with the extrapolation
//   rows (normal LAST); y = (V^T x V^T x V^T) (sum_q Dc_q^T x^(q) + W c u + lifts).
// Each thread writes only its own cell's y block (owner computes).
#pragma once
#include "dg_cell.cuh"
#include "dg_gen.cuh"

namespace dg {

#ifndef DG_REG_NMAX
#define DG_REG_NMAX 3      // constant diagonal D (fast path)
#endif
#ifndef DG_REG_GMAX
#define DG_REG_GMAX 3      // full / per-cell tensors (general path; n = 3 spills ~0.5 KB and still wins 1.7x)
#endif

// full 1D tables of the register kernel (tables.cpp): V_ij = theta_j(xi_i), G_ij = theta'_j(xi_i),
// Dc = G V^-1 (the
// collocation derivative), Gauss weights, the Lagrange rows L_l(0), L_l(1), L'_l(0), L'_l(1)
// and theta_j(0), theta_j(1), theta'_j(0), theta'_j(1)
template <int N>
struct RTab {
    double V[N][N], G[N][N], Dc[N][N], w[N], L[4][N], th0[N], th1[N], dth0[N], dth1[N];
};
__constant__ RTab<DG_N> g_rtab;

// index of (e along axis D, (a, b) on the other two axes in increasing order)
template <int N, int D>
__host__ __device__ __forceinline__ constexpr int rat(int e, int a, int b)
{
    return D == 0 ? e + N * (a + N * b) : (D == 1 ? a + N * (e + N * b) : a + N * (b + N * e));
}

// o(i along D) = sum_j M[i][j] a(j along D)
template <int N, int D>
__device__ __forceinline__ void rcontract(const double (&M)[N][N], const double (&a)[N * N * N], double (&o)[N * N * N])
{
#pragma unroll
    for (int b = 0; b < N; ++b)
#pragma unroll
        for (int c = 0; c < N; ++c)
#pragma unroll
            for (int i = 0; i < N; ++i) {
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) acc = fma(M[i][j], a[rat<N, D>(j, b, c)], acc);
                o[rat<N, D>(i, b, c)] = acc;
            }
}

// o(j along D) = sum_i M[i][j] a(i along D)   (transposed stage)
template <int N, int D>
__device__ __forceinline__ void rcontract_t(const double (&M)[N][N], const double (&a)[N * N * N], double (&o)[N * N * N])
{
#pragma unroll
    for (int b = 0; b < N; ++b)
#pragma unroll
        for (int c = 0; c < N; ++c)
#pragma unroll
            for (int j = 0; j < N; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int i = 0; i < N; ++i) acc = fma(M[i][j], a[rat<N, D>(i, b, c)], acc);
                o[rat<N, D>(j, b, c)] = acc;
            }
}

// the neighbour block across face f = 2q + s inside this rank's z (local or periodic wrap), as
// nb_load resolves it; a neighbour on another rank is read from the trace halo (reg_ghost)
template <int N>
__device__ __forceinline__ const double* reg_nb(const KParams& p, const double* zc, int64_t n3, const int (&lc)[3],
                                                int q, int s)
{
    const int lq = lc[q];
    const int nq = (int)p.nloc[q];
    const int64_t st = (q == 0) ? 1 : (q == 1) ? p.nloc[0] : p.nloc[0] * p.nloc[1];
    const int64_t wst = (int64_t)(nq - 1) * st * n3;
    const double* zn = s == 0 ? ((lq > 0) ? zc - st * n3 : zc + wst) : ((lq + 1 < nq) ? zc + st * n3 : zc - wst);
#ifdef DG_CHECK
    {
        const int64_t nall = p.nloc[0] * p.nloc[1] * p.nloc[2] * n3;
        DG_ASSERT(zn >= p.z && zn + n3 <= p.z + nall);
    }
#endif
    return zn;
}
// the normal-first contraction [u | d] (2 n^2) of the other-rank neighbour across face 2q + s
// (dg_trace_pack), or nullptr when that neighbour is in this rank's z
template <int N>
__device__ __forceinline__ const double* reg_ghost(const KParams& p, const int (&lc)[3], int q, int s)
{
    const int lq = lc[q];
    const int nq = (int)p.nloc[q];
    if (p.wrap[q] || (s == 0 ? lq > 0 : lq + 1 < nq)) return nullptr;
    const int64_t gi = (q == 0) ? (lc[1] + p.nloc[1] * lc[2]) : (q == 1) ? (lc[0] + p.nloc[0] * lc[2])
                                                                        : (lc[0] + p.nloc[0] * lc[1]);
    DG_ASSERT(p.ghost[2 * q + s] != nullptr);
    return p.ghost[2 * q + s] + gi * 2 * N * N;
}

template <int N>
__device__ __forceinline__ void reg_load(const double* src, double (&a)[N * N * N])
{
    constexpr int N3 = N * N * N;
    if constexpr (N3 % 2 == 0) {
#pragma unroll
        for (int e = 0; e < N3; e += 2) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(src + e));
            a[e] = v.x;
            a[e + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < N3; ++e) a[e] = __ldg(src + e);
    }
}

// ---------------------------------------------------------------------------------- staged blocks (n = 3)
// One thread per cell and 128 consecutive cells per CTA: the CTA's own blocks (with the x-neighbours
// at both ends of the range) and the rows of y-neighbour blocks below and above are contiguous
// ranges of z, so they arrive by three bulk copies (cp.async.bulk) into linear shared-memory images
// and y leaves by one, instead of 27 strided 8-byte loads / stores per block and thread (ncu C4-k2:
// long_scoreboard and lg_throttle were the top stalls at 26 % issue). A neighbour outside the images
// (periodic wrap, another rank, the z direction) is read from global memory as before.
#ifndef DG_REG_STAGE
#define DG_REG_STAGE 4     // bit 2 (n - 2) + GEN: staged instantiations (bit 2: n = 3, constant diagonal D)
#endif
constexpr int REG_CTA = 128;                       // threads = cells per CTA of dg_reg_kernel
template <int N, bool GEN> struct RStage {
    static constexpr bool ON = N >= 2 && N <= 3 && ((DG_REG_STAGE >> (2 * (N - 2) + (GEN ? 1 : 0))) & 1);
    static constexpr int N3 = N * N * N;
    static constexpr int IMG0 = (REG_CTA + 2) * N3 + 2;   // own blocks + one x-neighbour each side (+ shift pad)
    static constexpr int IMG = REG_CTA * N3 + 2;          // one row of y-neighbour blocks
#ifndef DG_REG_NIMG
#define DG_REG_NIMG 1      // 1: the own / x image only (C4-k2 68.9 against 68.5 GDOF/s with the y rows too)
#endif
    static constexpr int NIMG = DG_REG_NIMG;
    static constexpr int MB = IMG0 + (NIMG > 1 ? 2 * IMG : 0);   // the mbarrier (doubles)
    static constexpr int BYTES = ON ? MB * 8 + 16 : 0;
};
struct RImg {
    const double* S;   // smem: global double d of the range sits at S[d - d0]
    int64_t d0, d1;    // global double range [d0, d1) of z held (empty: d0 == d1)
};
// tid 0: bulk-copy the 16-byte-aligned interior of z[d0, d1) to base + (d0 & 1) + ..., plain loads for an
// odd leading / trailing double (stored after the wait by the caller's thread 0, see rimg_fix)
__device__ __forceinline__ RImg rimg_make(double* base, int64_t d0, int64_t d1)
{
    RImg im;
    im.d0 = d0;
    im.d1 = d1 > d0 ? d1 : d0;
    im.S = base + (d0 & 1);                        // S + (d - d0) == z + d (mod 16 bytes)
    return im;
}
__device__ __forceinline__ uint32_t rimg_bytes(const RImg& im)
{
    const int64_t a0 = im.d0 + (im.d0 & 1), a1 = im.d1 - (im.d1 & 1);
    return a1 > a0 ? (uint32_t)((a1 - a0) * 8) : 0u;
}
__device__ __forceinline__ void rimg_issue(const double* z, const RImg& im, uint64_t* mbar)
{
    const int64_t a0 = im.d0 + (im.d0 & 1);
    const uint32_t b = rimg_bytes(im);
    if (b) bulk::load(const_cast<double*>(im.S) + (a0 - im.d0), z + a0, b, mbar);
}
__device__ __forceinline__ void rimg_fix(const double* z, const RImg& im)
{
    double* S = const_cast<double*>(im.S);
    if (im.d1 <= im.d0) return;
    if (im.d0 & 1) S[0] = __ldg(z + im.d0);                                  // odd leading double
    if (im.d1 & 1) S[im.d1 - 1 - im.d0] = __ldg(z + im.d1 - 1);              // odd trailing double
}
template <int N>
__device__ __forceinline__ void reg_load_smem(const double* src, double (&a)[N * N * N])
{
#pragma unroll
    for (int e = 0; e < N * N * N; ++e) a[e] = src[e];
}

// 2D face-array stages: o(i, b) = sum_j M[i][j] a(j, b) (AX = 0) or o(a, i) = sum_j M[i][j] a(a, j)
template <int N, int AX, bool TR>
__device__ __forceinline__ void fstage(const double (&M)[N][N], const double (&a)[N][N], double (&o)[N][N])
{
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < N; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double m = TR ? M[j][i] : M[i][j];
                acc = fma(m, AX == 0 ? a[j][c] : a[c][j], acc);
            }
            if (AX == 0) o[i][c] = acc;
            else o[c][i] = acc;
        }
}

// the faces of direction Q: own traces, neighbour traces, fluxes, lifts into X (quadrature space).
// GEN: full per-cell tensors (dg_gen.cuh semantics): nu.D grad u with the tangential derivatives
// of both traces (own: Dc along the face lines; neighbour: G in its tangential stages), weights
// w-+ = d+-/(d- + d+), penalty <d-, d+> sigma_q (C-5), tangential test-derivative lifts with Dc^T.
template <int N, int Q, bool GEN, bool GH>
__device__ __forceinline__ void reg_faces(const KParams& p, const RTab<N>& R, const double* zc, int64_t n3,
                                          const int (&lc)[3], int64_t cell, unsigned nbmask, bool do_int, bool do_bnd,
                                          const double (&Dw)[6], const double (&u)[N * N * N], double (&X)[N * N * N],
                                          const double* slo = nullptr, const double* shi = nullptr)
{
    constexpr int T1 = (Q == 0) ? 1 : 0, T2 = (Q == 2) ? 1 : 2;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const bool interior = (nbmask >> (2 * Q + s)) & 1u;
        if (interior ? !do_int : !do_bnd) continue;
        double un[N][N], sn[N][N];                 // neighbour u+ and nu.D+ grad u+ (physical)
        double dnb = 0.0;                          // neighbour D_qq (GEN)
        if (interior) {
            // normal first: the neighbour is seen at its x_q = 1 (s = 0) or 0 (s = 1)
            double cu[N][N], cd[N][N];
            if (const double* tr = GH ? reg_ghost<N>(p, lc, Q, s) : nullptr) {   // contracted by its rank
#pragma unroll
                for (int a = 0; a < N; ++a)
#pragma unroll
                    for (int b = 0; b < N; ++b) {
                        cu[a][b] = __ldg(tr + a + N * b);
                        cd[a][b] = __ldg(tr + N * N + a + N * b);
                    }
            } else {
                double zn[N * N * N];
                if (const double* sb = s ? shi : slo) reg_load_smem<N>(sb, zn);   // staged image (RStage)
                else reg_load<N>(reg_nb<N>(p, zc, n3, lc, Q, s), zn);
#pragma unroll
                for (int a = 0; a < N; ++a)
#pragma unroll
                    for (int b = 0; b < N; ++b) {
                        double su = 0.0, sd = 0.0;
#pragma unroll
                        for (int e = 0; e < N; ++e) {
                            const double v = zn[rat<N, Q>(e, a, b)];
                            su = fma(s ? R.th0[e] : R.th1[e], v, su);
                            sd = fma(s ? R.dth0[e] : R.dth1[e], v, sd);
                        }
                        cu[a][b] = su;
                        cd[a][b] = sd;
                    }
            }
            // tangential stages: V along the first, then the second tangential axis
            double t0[N][N], t1[N][N], dn[N][N];
            fstage<N, 0, false>(R.V, cu, t0);
            fstage<N, 1, false>(R.V, t0, un);
            fstage<N, 0, false>(R.V, cd, t1);
            fstage<N, 1, false>(R.V, t1, dn);
            if constexpr (GEN) {
                const double* Dn = nb_dfield(p, lc, cell, 2 * Q + s, nbmask);
                dnb = __ldg(Dn + Q);
                const double cqq = dnb * p.hinv[Q], cq1 = __ldg(Dn + dsym(Q, T1)) * p.hinv[T1],
                             cq2 = __ldg(Dn + dsym(Q, T2)) * p.hinv[T2];
                double g1[N][N], g2[N][N];
                fstage<N, 0, false>(R.G, cu, t1);          // d/dt1: G along the first axis, V along the second
                fstage<N, 1, false>(R.V, t1, g1);
                fstage<N, 1, false>(R.G, t0, g2);          // d/dt2: V along the first, G along the second
#pragma unroll
                for (int a = 0; a < N; ++a)
#pragma unroll
                    for (int b = 0; b < N; ++b) sn[a][b] = fma(cqq, dn[a][b], fma(cq1, g1[a][b], cq2 * g2[a][b]));
            } else {
#pragma unroll
                for (int a = 0; a < N; ++a)
#pragma unroll
                    for (int b = 0; b < N; ++b) sn[a][b] = p.Dqq_h[Q] * dn[a][b];
            }
        }
        // own traces by extrapolation of the Gauss-point values along the normal
        double uo[N][N], dref[N][N];
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) {
                double su = 0.0, sd = 0.0;
#pragma unroll
                for (int e = 0; e < N; ++e) {
                    const double v = u[rat<N, Q>(e, a, b)];
                    su = fma(R.L[s][e], v, su);
                    sd = fma(R.L[2 + s][e], v, sd);
                }
                uo[a][b] = su;
                dref[a][b] = sd;
            }
        double cvf[N][N], cgf[N][N];               // value and normal-derivative lift coefficients
        if constexpr (GEN) {
            const double dme = Dw[Q];
            const double cn = dme * p.hinv[Q], c1 = Dw[dsym(Q, T1)] * p.hinv[T1], c2 = Dw[dsym(Q, T2)] * p.hinv[T2];
            double d1[N][N], d2[N][N];
            fstage<N, 0, false>(R.Dc, uo, d1);           // tangential derivatives of the own trace
            fstage<N, 1, false>(R.Dc, uo, d2);
            const double dm = s ? dme : dnb, dp = s ? dnb : dme;      // delta of T-, T+
            const double dsum = dm + dp;
            const double rsum = dsum == 0.0 ? 0.0 : 1.0 / dsum;
            const double wm = dsum == 0.0 ? 0.5 : dp * rsum, wp = dsum == 0.0 ? 0.5 : dm * rsum;   // C-5
            const double gam = (interior ? 2.0 * dm * dp * rsum : dme) * p.sigq[Q];
            const double wself = s ? wm : wp;
            const double bq = p.bq[Q];
            double f1[N][N], f2[N][N];
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int b = 0; b < N; ++b) {
                    const double Wf = p.dF[Q] * R.w[a] * R.w[b];
                    const double so = fma(cn, dref[a][b], fma(c1, d1[a][b], c2 * d2[a][b]));
                    double coef;
                    if (interior) {
                        const double um = s ? uo[a][b] : un[a][b], up = s ? un[a][b] : uo[a][b];
                        const double sm = s ? so : sn[a][b], sp = s ? sn[a][b] : so;
                        const double Phi = (bq >= 0.0) ? bq * um : bq * up;   // upwind flux
                        const double J = um - up;
                        const double com = Phi - (wm * sm + wp * sp) + gam * J;
                        cvf[a][b] = s ? Wf * com : -Wf * com;
                        coef = -Wf * wself * J;
                    } else {
                        const double nu = s ? 1.0 : -1.0;                      // outward normal
                        const double bn = nu * bq;
                        const double Phi = (bn >= 0.0) ? bn * uo[a][b] : 0.0;
                        cvf[a][b] = Wf * (Phi - nu * so + gam * uo[a][b]);
                        coef = -Wf * uo[a][b] * nu;
                    }
                    cgf[a][b] = coef * cn;                                     // normal part (L')
                    f1[a][b] = coef * c1;                                      // tangential parts (Dc^T)
                    f2[a][b] = coef * c2;
                }
            double l1[N][N], l2[N][N];
            fstage<N, 0, true>(R.Dc, f1, l1);
            fstage<N, 1, true>(R.Dc, f2, l2);
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int b = 0; b < N; ++b) cvf[a][b] += l1[a][b] + l2[a][b];
        } else {
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int b = 0; b < N; ++b) {
                    const double Wf = p.dF[Q] * R.w[a] * R.w[b];
                    const FaceOut fo = interior ? flux_interior(p, Q, s, Wf, uo[a][b], dref[a][b], un[a][b], sn[a][b])
                                                : flux_boundary(p, Q, s, Wf, uo[a][b], dref[a][b]);
                    cvf[a][b] = fo.cv;
                    cgf[a][b] = fo.cg;
                }
        }
        // lift (normal direction LAST) into the quadrature-space accumulator
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b)
#pragma unroll
                for (int e = 0; e < N; ++e) {
                    const int ix = rat<N, Q>(e, a, b);
                    X[ix] = fma(cvf[a][b], R.L[s][e], fma(cgf[a][b], R.L[2 + s][e], X[ix]));
                }
    }
}

// minimum CTAs per SM: n = 2 at 5 with constant D (96 registers: C4-k1 83.3 -> 84.7 GDOF/s) and
// at 4 with tensors (128 registers, a few spills instead of 150: Problem A k = 1 47.2 -> 50.9)
#ifndef DG_RMINB3
#define DG_RMINB3 1
#endif
#ifndef DG_RMINB2F
#define DG_RMINB2F 5
#endif
#ifndef DG_RMINB
#define DG_RMINB(n, gen) ((n) == 2 ? ((gen) ? 4 : DG_RMINB2F) : DG_RMINB3)
#endif
template <int N, bool GEN, bool GH = false>
__global__ void __launch_bounds__(REG_CTA, DG_RMINB(N, GEN)) dg_reg_kernel(const __grid_constant__ KParams p)
{
    constexpr int N3 = N * N * N;
    const RTab<N>& R = g_rtab;
    int64_t task = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // staged images (RStage): consecutive tasks are consecutive cells when the task box spans whole
    // x-rows and y-planes of this rank's box
    const bool stg = RStage<N, GEN>::ON && p.tma == 2 && !p.task_list && p.task_lo[0] == 0 && p.task_lo[1] == 0 &&
                     p.task_cnt[0] == p.nloc[0] && p.task_cnt[1] == p.nloc[1];
    const bool valid = task < p.ntasks;
    if (!stg && !valid) return;
    if (!valid) task = p.ntasks - 1;               // (staged: every thread takes part in the barriers)
    extern __shared__ __align__(16) double rsm[];
    int64_t soff[3] = {0, 0, 0};                   // first global double of each image
    if constexpr (RStage<N, GEN>::ON) {
        if (stg) {
            const int64_t nxy = p.nloc[0] * p.nloc[1], ncell = nxy * p.nloc[2];
            const int64_t cb = p.task_lo[2] * nxy + blockIdx.x * (int64_t)REG_CTA;    // first cell of the CTA
            const int64_t nv = min((int64_t)REG_CTA, p.ntasks - blockIdx.x * (int64_t)REG_CTA);
            auto clampc = [&](int64_t c) { return c < 0 ? (int64_t)0 : (c > ncell ? ncell : c); };
            const int64_t lo[3] = {clampc(cb - 1), clampc(cb - p.nloc[0]), clampc(cb + p.nloc[0])};
            // (RStage::NIMG = 1: the own / x image only, the y-neighbour rows from global memory)
            const int64_t hi[3] = {clampc(cb + nv + 1), RStage<N, GEN>::NIMG > 1 ? clampc(cb - p.nloc[0] + nv) : lo[1],
                                   RStage<N, GEN>::NIMG > 1 ? clampc(cb + p.nloc[0] + nv) : lo[2]};
#pragma unroll
            for (int i = 0; i < 3; ++i) soff[i] = N3 * lo[i];
            uint64_t* mbar = reinterpret_cast<uint64_t*>(rsm + RStage<N, GEN>::MB);
            if (threadIdx.x == 0) {
                RImg im[3];
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    im[i] = rimg_make(rsm + (i == 0 ? 0 : RStage<N, GEN>::IMG0 + (i - 1) * RStage<N, GEN>::IMG), N3 * lo[i], N3 * hi[i]);
                tma::mbar_init_n(mbar, 1);
                tma::expect_tx(mbar, rimg_bytes(im[0]) + rimg_bytes(im[1]) + rimg_bytes(im[2]));
#pragma unroll
                for (int i = 0; i < 3; ++i) rimg_issue(p.z, im[i], mbar);
#pragma unroll
                for (int i = 0; i < 3; ++i) rimg_fix(p.z, im[i]);
            }
            __syncthreads();
            tma::wait(mbar, 0);
        }
    }
    int lc[3];
    if (p.task_list) {
        const int64_t e = p.task_list[task];
        lc[0] = (int)(e % p.nloc[0]);
        lc[1] = (int)((e / p.nloc[0]) % p.nloc[1]);
        lc[2] = (int)(e / (p.nloc[0] * p.nloc[1]));
    } else {                                       // lexicographic in the task box (x fastest)
        const int64_t cx = p.task_cnt[0], cy = p.task_cnt[1];
        lc[0] = (int)(p.task_lo[0] + task % cx);
        lc[1] = (int)(p.task_lo[1] + (task / cx) % cy);
        lc[2] = (int)(p.task_lo[2] + task / (cx * cy));
    }
    const int64_t n3 = N3;
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

    // this thread's blocks in the staged images: own, x- / y-neighbours inside this rank's box (no wrap)
    const double *sown = nullptr, *sx0 = nullptr, *sx1 = nullptr, *sy0 = nullptr, *sy1 = nullptr;
    if constexpr (RStage<N, GEN>::ON) {
        if (stg) {
            const double* S0 = rsm + (soff[0] & 1);
            const double* S1 = rsm + RStage<N, GEN>::IMG0 + (soff[1] & 1);
            const double* S2 = rsm + RStage<N, GEN>::IMG0 + RStage<N, GEN>::IMG + (soff[2] & 1);
            sown = S0 + (cell * n3 - soff[0]);
            if (lc[0] > 0) sx0 = sown - n3;
            if (lc[0] + 1 < p.nloc[0]) sx1 = sown + n3;
            if (RStage<N, GEN>::NIMG > 1 && lc[1] > 0) sy0 = S1 + ((cell - p.nloc[0]) * n3 - soff[1]);
            if (RStage<N, GEN>::NIMG > 1 && lc[1] + 1 < p.nloc[1]) sy1 = S2 + ((cell + p.nloc[0]) * n3 - soff[2]);
            constexpr int IMG0 = RStage<N, GEN>::IMG0;   // (the staged blocks lie inside image 0)
            DG_ASSERT(sown >= rsm && sown + n3 <= rsm + IMG0);
            DG_ASSERT(!sx0 || (sx0 >= rsm && sx0 + n3 <= rsm + IMG0));
            DG_ASSERT(!sx1 || (sx1 >= rsm && sx1 + n3 <= rsm + IMG0));
        }
    }
    double u[N3], t[N3], X[N3];
    if (sown) reg_load_smem<N>(sown, t);
    else reg_load<N>(zc, t);
    rcontract<N, 0>(R.V, t, u);
    rcontract<N, 1>(R.V, u, t);
    rcontract<N, 2>(R.V, t, u);                     // u at the Gauss points
#pragma unroll
    for (int i = 0; i < N3; ++i) X[i] = 0.0;
    double Dw[6] = {0, 0, 0, 0, 0, 0};
    if constexpr (GEN) {
#pragma unroll
        for (int i = 0; i < 6; ++i) Dw[i] = __ldg(p.Dfield + 6 * cell + i);
    }
    if (do_vol) {
        if constexpr (GEN && N >= 3) {
            // as below, with the reference derivatives recomputed per role (two arrays live instead
            // of four: registers)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double kb = p.dT * p.kb[q];
#pragma unroll
                for (int i = 0; i < N3; ++i) t[i] = -kb * u[i];
#pragma unroll
                for (int sd = 0; sd < 3; ++sd) {
                    double g[N3];
                    if (sd == 0) rcontract<N, 0>(R.Dc, u, g);
                    else if (sd == 1) rcontract<N, 1>(R.Dc, u, g);
                    else rcontract<N, 2>(R.Dc, u, g);
                    const double dh = p.dT * Dw[dsym(q, sd)] * (p.hinv[q] * p.hinv[sd]);
#pragma unroll
                    for (int i = 0; i < N3; ++i) t[i] = fma(dh, g[i], t[i]);
                }
#pragma unroll
                for (int iz = 0; iz < N; ++iz)
#pragma unroll
                    for (int iy = 0; iy < N; ++iy)
#pragma unroll
                        for (int ix = 0; ix < N; ++ix) {
                            const int i = ix + N * (iy + N * iz);
                            t[i] *= R.w[ix] * R.w[iy] * R.w[iz];
                        }
                double o[N3];
                if (q == 0) rcontract_t<N, 0>(R.Dc, t, o);
                else if (q == 1) rcontract_t<N, 1>(R.Dc, t, o);
                else rcontract_t<N, 2>(R.Dc, t, o);
#pragma unroll
                for (int i = 0; i < N3; ++i) X[i] += o[i];
            }
        } else if constexpr (GEN) {
            // x^(r) = W (sum_s D_rs/(h_r h_s) d_s u - b_r/h_r u), X += Dc_r^T x^(r)   (eq:gauss_points)
            double g0[N3], g1[N3], g2[N3];
            rcontract<N, 0>(R.Dc, u, g0);
            rcontract<N, 1>(R.Dc, u, g1);
            rcontract<N, 2>(R.Dc, u, g2);
            double Dh[3][3];
#pragma unroll
            for (int rr = 0; rr < 3; ++rr)
#pragma unroll
                for (int ss = 0; ss < 3; ++ss) Dh[rr][ss] = p.dT * Dw[dsym(rr, ss)] * (p.hinv[rr] * p.hinv[ss]);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double kb = p.dT * p.kb[q];
#pragma unroll
                for (int iz = 0; iz < N; ++iz)
#pragma unroll
                    for (int iy = 0; iy < N; ++iy)
#pragma unroll
                        for (int ix = 0; ix < N; ++ix) {
                            const int i = ix + N * (iy + N * iz);
                            const double W = R.w[ix] * R.w[iy] * R.w[iz];
                            t[i] = W * (Dh[q][0] * g0[i] + Dh[q][1] * g1[i] + Dh[q][2] * g2[i] - kb * u[i]);
                        }
                double o[N3];
                if (q == 0) rcontract_t<N, 0>(R.Dc, t, o);
                else if (q == 1) rcontract_t<N, 1>(R.Dc, t, o);
                else rcontract_t<N, 2>(R.Dc, t, o);
#pragma unroll
                for (int i = 0; i < N3; ++i) X[i] += o[i];
            }
        } else {
            // roles: X += Dc_q^T x^(q), x^(q) = W (D_qq/h_q^2 d_q u - b_q/h_q u)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (q == 0) rcontract<N, 0>(R.Dc, u, t);
                else if (q == 1) rcontract<N, 1>(R.Dc, u, t);
                else rcontract<N, 2>(R.Dc, u, t);
                const double kd = p.dT * p.Dhat[4 * q], kb = p.dT * p.kb[q];
#pragma unroll
                for (int iz = 0; iz < N; ++iz)
#pragma unroll
                    for (int iy = 0; iy < N; ++iy)
#pragma unroll
                        for (int ix = 0; ix < N; ++ix) {
                            const int i = ix + N * (iy + N * iz);
                            const double W = R.w[ix] * R.w[iy] * R.w[iz];
                            t[i] = W * fma(kd, t[i], -kb * u[i]);
                        }
                double o[N3];
                if (q == 0) rcontract_t<N, 0>(R.Dc, t, o);
                else if (q == 1) rcontract_t<N, 1>(R.Dc, t, o);
                else rcontract_t<N, 2>(R.Dc, t, o);
#pragma unroll
                for (int i = 0; i < N3; ++i) X[i] += o[i];
            }
        }
        const double wc = p.dT * p.c;          // reaction W c u
#pragma unroll
        for (int iz = 0; iz < N; ++iz)
#pragma unroll
            for (int iy = 0; iy < N; ++iy)
#pragma unroll
                for (int ix = 0; ix < N; ++ix) {
                    const int i = ix + N * (iy + N * iz);
                    X[i] = fma(wc * R.w[ix] * R.w[iy] * R.w[iz], u[i], X[i]);
                }
    }
    reg_faces<N, 0, GEN, GH>(p, R, zc, n3, lc, cell, nbmask, do_int, do_bnd, Dw, u, X, sx0, sx1);
    reg_faces<N, 1, GEN, GH>(p, R, zc, n3, lc, cell, nbmask, do_int, do_bnd, Dw, u, X, sy0, sy1);
    reg_faces<N, 2, GEN, GH>(p, R, zc, n3, lc, cell, nbmask, do_int, do_bnd, Dw, u, X);
    rcontract_t<N, 2>(R.V, X, t);
    rcontract_t<N, 1>(R.V, t, u);
    rcontract_t<N, 0>(R.V, u, t);                   // y block
    double* yc = p.y + cell * n3;
    if constexpr (RStage<N, GEN>::ON) {
        if (stg && p.epi == 0) {   // y through a linear image (over the free images) and one bulk store
            const int64_t nv = min((int64_t)REG_CTA, p.ntasks - blockIdx.x * (int64_t)REG_CTA);
            const int64_t cb = cell - threadIdx.x;
            const int64_t d0 = cb * n3, d1 = (cb + nv) * n3;
            __syncthreads();                           // every image read
            double* S = rsm + (d0 & 1);                // S + (d - d0) == y + d (mod 16 bytes)
            if (valid) {
#pragma unroll
                for (int e = 0; e < N3; ++e) S[threadIdx.x * N3 + e] = t[e];
            }
            tma::fence_async();
            __syncthreads();
            const int64_t a0 = d0 + (d0 & 1), a1 = d1 - (d1 & 1);
            if (threadIdx.x == 0) {
                if (a1 > a0) bulk::store(p.y + a0, S + (a0 - d0), (uint32_t)((a1 - a0) * 8));
                if (d0 & 1) __stcs(p.y + d0, S[0]);
                if (d1 & 1) __stcs(p.y + d1 - 1, S[d1 - 1 - d0]);
            }
            return;
        }
    }
    if (!valid) return;
    epilogue<N3>(p, cell * n3, t);
    if constexpr (N3 % 2 == 0) {
#pragma unroll
        for (int e = 0; e < N3; e += 2) __stcs(reinterpret_cast<double2*>(yc + e), make_double2(t[e], t[e + 1]));
    } else {
#pragma unroll
        for (int e = 0; e < N3; ++e) __stcs(yc + e, t[e]);
    }
}

}  // namespace dg
