// Register-resident cell kernel for the smallest bases (constant diagonal D; the fast path of
// dg_cell.cuh for n <= DG_REG_NMAX): one THREAD per cell, the whole n^3 block and every
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

namespace dg {

#ifndef DG_REG_NMAX
#define DG_REG_NMAX 3
#endif

// full 1D tables of the register kernel (tables.cpp): V_ij = theta_j(xi_i), Dc = G V^-1 (the
// collocation derivative), Gauss weights, the Lagrange rows L_l(0), L_l(1), L'_l(0), L'_l(1)
// and theta_j(0), theta_j(1), theta'_j(0), theta'_j(1)
template <int N>
struct RTab {
    double V[N][N], Dc[N][N], w[N], L[4][N], th0[N], th1[N], dth0[N], dth1[N];
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

// the neighbour block across face f = 2q + s (nullptr: none), as nb_load resolves it
template <int N>
__device__ __forceinline__ const double* reg_nb(const KParams& p, const double* zc, int64_t n3, const int (&lc)[3],
                                                int q, int s, unsigned nbmask)
{
    if (!((nbmask >> (2 * q + s)) & 1u)) return nullptr;
    const int lq = lc[q];
    const int nq = (int)p.nloc[q];
    const int64_t st = (q == 0) ? 1 : (q == 1) ? p.nloc[0] : p.nloc[0] * p.nloc[1];
    const int64_t gi = (q == 0) ? (lc[1] + p.nloc[1] * lc[2]) : (q == 1) ? (lc[0] + p.nloc[0] * lc[2])
                                                                        : (lc[0] + p.nloc[0] * lc[1]);
    const int64_t wst = (int64_t)(nq - 1) * st * n3;
    if (s == 0) return (lq > 0) ? zc - st * n3 : (p.wrap[q] ? zc + wst : p.ghost[2 * q] + gi * n3);
    return (lq + 1 < nq) ? zc + st * n3 : (p.wrap[q] ? zc - wst : p.ghost[2 * q + 1] + gi * n3);
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

// the faces of direction Q: own traces, neighbour traces, fluxes, lifts into X (quadrature space)
template <int N, int Q>
__device__ __forceinline__ void reg_faces(const KParams& p, const RTab<N>& R, const double* zc, int64_t n3,
                                          const int (&lc)[3], unsigned nbmask, bool do_int, bool do_bnd,
                                          const double (&u)[N * N * N], double (&X)[N * N * N])
{
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const bool interior = (nbmask >> (2 * Q + s)) & 1u;
        if (interior ? !do_int : !do_bnd) continue;
        double un[N][N], dn[N][N];
        if (interior) {
            double zn[N * N * N];
            reg_load<N>(reg_nb<N>(p, zc, n3, lc, Q, s, nbmask), zn);
            // normal first: the neighbour is seen at its x_q = 1 (s = 0) or 0 (s = 1)
            double cu[N][N], cd[N][N];
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
            // V along the first, then the second tangential axis
            double tu[N][N], td[N][N];
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int b = 0; b < N; ++b) {
                    double su = 0.0, sd = 0.0;
#pragma unroll
                    for (int j = 0; j < N; ++j) {
                        su = fma(R.V[i][j], cu[j][b], su);
                        sd = fma(R.V[i][j], cd[j][b], sd);
                    }
                    tu[i][b] = su;
                    td[i][b] = sd;
                }
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    double su = 0.0, sd = 0.0;
#pragma unroll
                    for (int j = 0; j < N; ++j) {
                        su = fma(R.V[i][j], tu[a][j], su);
                        sd = fma(R.V[i][j], td[a][j], sd);
                    }
                    un[a][i] = su;
                    dn[a][i] = sd;
                }
        }
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) {
                // own traces by extrapolation of the Gauss-point values along the normal
                double uo = 0.0, dref = 0.0;
#pragma unroll
                for (int e = 0; e < N; ++e) {
                    const double v = u[rat<N, Q>(e, a, b)];
                    uo = fma(R.L[s][e], v, uo);
                    dref = fma(R.L[2 + s][e], v, dref);
                }
                const double Wf = p.dF[Q] * R.w[a] * R.w[b];
                const FaceOut fo = interior ? flux_interior(p, Q, s, Wf, uo, dref, un[a][b], p.Dqq_h[Q] * dn[a][b])
                                            : flux_boundary(p, Q, s, Wf, uo, dref);
#pragma unroll
                for (int e = 0; e < N; ++e) {
                    const int ix = rat<N, Q>(e, a, b);
                    X[ix] = fma(fo.cv, R.L[s][e], fma(fo.cg, R.L[2 + s][e], X[ix]));
                }
            }
    }
}

#ifdef DG_RMINB
#define DG_REG_BOUNDS __launch_bounds__(128, DG_RMINB)
#else
#define DG_REG_BOUNDS __launch_bounds__(128)
#endif
template <int N>
__global__ void DG_REG_BOUNDS dg_reg_kernel(const __grid_constant__ KParams p)
{
    constexpr int N3 = N * N * N;
    const RTab<N>& R = g_rtab;
    const int64_t task = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (task >= p.ntasks) return;
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

    double u[N3], t[N3], X[N3];
    reg_load<N>(zc, t);
    rcontract<N, 0>(R.V, t, u);
    rcontract<N, 1>(R.V, u, t);
    rcontract<N, 2>(R.V, t, u);                     // u at the Gauss points
#pragma unroll
    for (int i = 0; i < N3; ++i) X[i] = 0.0;
    if (do_vol) {
        // roles: X += Dc_q^T x^(q), x^(q) = W (D_qq/h_q^2 d_q u - b_q/h_q u); reaction W c u
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
        const double wc = p.dT * p.c;
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
    reg_faces<N, 0>(p, R, zc, n3, lc, nbmask, do_int, do_bnd, u, X);
    reg_faces<N, 1>(p, R, zc, n3, lc, nbmask, do_int, do_bnd, u, X);
    reg_faces<N, 2>(p, R, zc, n3, lc, nbmask, do_int, do_bnd, u, X);
    rcontract_t<N, 2>(R.V, X, t);
    rcontract_t<N, 1>(R.V, t, u);
    rcontract_t<N, 0>(R.V, u, t);                   // y block
    double* yc = p.y + cell * n3;
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
