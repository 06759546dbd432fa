// Fused cell kernel: y = A z for the SIPG/WSIPG operator of arXiv 1711.10885,
// FP64, sm_100a. One CTA processes C cells; each cell is worked on by n^2
// threads, each thread owning one "pencil" (a line of n points along one
// direction) in each of three roles (x-, y- and z-pencil).
//
// Per cell (Algorithm 1, reorganised owner-computes):
//   (1) evaluate u at the n^3 Gauss points by sum factorization
//       u_q = (V x V x V) z              (eq:evalfe; kernel eq:sum_fact_kernel :590-595)
//       and the reference gradient by collocation derivatives along each pencil
//       (Dc = G V^{-1}, exact since u in Q_k: DESIGN.md "What differs")
//   (2) quadrature-point data x^(r) (eq:gauss_points) and x^(0) = c u W
//   (3) integrate: y = (V^T x V^T x V^T)(x^(0) + sum_r Dc_r^T x^(r) + face lifts)   (eq:evalblf, :425-444)
//   (4-10) faces: own traces (u, normal derivative) are 1D extrapolations of u_q along the
//       normal (L_l(s), L'_l(s)); neighbour traces are the paper's face sum factorization
//       with the normal direction FIRST: theta(s) / theta'(s) contraction of the
//       neighbour's coefficients, then V along the two tangential directions. The SIPG
//       consistency, symmetry, penalty and upwind terms (eq:blf :301-315, Phi :334-341) are
//       evaluated pointwise and lifted back with the normal direction LAST, into the
//       quadrature-space array before the transposed V stages. Each cell writes only its
//       own y block: no atomics, no races, y stored once.
#pragma once
#include "dg_internal.h"

namespace dg {

template <int N>
struct Tab {
    double V[N][N];
    double Dc[N][N];
    double w[N];
    double L0[N], L1[N], LD0[N], LD1[N];
    double th0[N], th1[N], dth0[N], dth1[N];
};

#ifndef DG_N
#error "dg_cell.cuh is compiled once per degree with -DDG_N=<k+1>"
#endif
// The 1D tables of this translation unit's degree (uploaded by upload_tables).
__constant__ Tab<DG_N> g_tab;

// Cells per CTA for each n (threads = C n^2; 2 CTAs per SM for n = 8).
template <int N> struct Cfg;
template <> struct Cfg<2>  { static constexpr int C = 32; };
template <> struct Cfg<3>  { static constexpr int C = 14; };
template <> struct Cfg<4>  { static constexpr int C = 8; };
template <> struct Cfg<5>  { static constexpr int C = 10; };
template <> struct Cfg<6>  { static constexpr int C = 7; };
template <> struct Cfg<7>  { static constexpr int C = 5; };
template <> struct Cfg<8>  { static constexpr int C = 4; };
template <> struct Cfg<9>  { static constexpr int C = 3; };
template <> struct Cfg<10> { static constexpr int C = 2; };
template <> struct Cfg<11> { static constexpr int C = 2; };

// Shared-memory layout of one n^3 cell array, chosen so that x-, y- and z-pencil
// accesses of a warp are (nearly) bank-conflict free (searched offline; n = 8 uses an
// XOR swizzle that is conflict free for all three access patterns).
template <int N> struct Lay {
    static constexpr int SY = (N == 6) ? 9 : (N == 10 ? 11 : N);
    static constexpr int SZ = (N == 2) ? 5 : (N == 3) ? 9 : (N == 4) ? 18 : (N == 5) ? 25 : (N == 6) ? 54
                            : (N == 7) ? 54 : (N == 9) ? 85 : (N == 10) ? 110 : 121;
    static constexpr int SLOT = (N == 2) ? 10 : (N == 3) ? 27 : (N == 4) ? 73 : (N == 5) ? 125 : (N == 6) ? 324
                              : (N == 7) ? 385 : (N == 9) ? 769 : (N == 10) ? 1100 : 1331;
    __device__ __forceinline__ static int at(int x, int y, int z) { return x + SY * y + SZ * z; }
};
template <> struct Lay<8> {
    static constexpr int SLOT = 512;
    __device__ __forceinline__ static int at(int x, int y, int z)
    {
        return (x ^ ((y >> 1) | ((z & 1) << 2))) + 8 * (y ^ (z & 1)) + 64 * z;
    }
};

// Face-trace arrays: 6 faces x 2 quantities x n^2 points, row padded.
template <int N> struct FLay {
    static constexpr int RS = N + 1;              // row stride
    static constexpr int ARR = N * RS + 1;        // one n x n array
    static constexpr int SLOT = 12 * ARR;
    __device__ __forceinline__ static int at(int arr, int i1, int i2) { return arr * ARR + i1 + RS * i2; }
};

template <int N>
struct Smem {
    static constexpr int C = Cfg<N>::C;
    static constexpr int PER_CELL = 3 * Lay<N>::SLOT + FLay<N>::SLOT;
    static constexpr int BYTES = C * PER_CELL * 8;
};

// out[i] = sum_j M[i][j] in[j]
template <int N>
__device__ __forceinline__ void mv(const double (&M)[N][N], const double* in, double* out)
{
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) s = fma(M[i][j], in[j], s);
        out[i] = s;
    }
}
// out[j] = sum_i M[i][j] in[i]
template <int N>
__device__ __forceinline__ void mtv(const double (&M)[N][N], const double* in, double* out)
{
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) s = fma(M[i][j], in[i], s);
        out[j] = s;
    }
}
template <int N>
__device__ __forceinline__ double dot(const double* a, const double* v)
{
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s = fma(a[i], v[i], s);
    return s;
}

// Face coefficient pair (cv, cgref) at one face point for a cell face in direction q,
// own side s (s = 1: face x_q = 1, this cell is T-; s = 0: face x_q = 0, this cell is T+).
//   uo, dref : own trace and reference normal derivative (d/dx_hat_q)
//   un, sn   : neighbour trace and physical normal flux D_qq d u/dx_q (nu = +e_q)
// Returns the contribution cv * phi_i + cg_phys * d_q phi_i as (cv, cgref = cg_phys / h_q).
struct FaceOut { double cv, cg; };

__device__ __forceinline__ FaceOut flux_interior(const KParams& p, int q, int s, double W, double uo, double dref,
                                                 double un, double sn)
{
    const double so = p.Dqq_h[q] * dref;           // D_qq du/dx_q
    const double um = s ? uo : un, up = s ? un : uo;
    const double sm = s ? so : sn, sp = s ? sn : so;
    const double bn = p.bq[q];
    const double Phi = (bn >= 0.0) ? bn * um : bn * up;       // upwind flux
    const double J = um - up;                                 // [[u]] = u- - u+
    const double Avg = 0.5 * (sm + sp);                       // {D grad u}_w . nu, w = 1/2 (constant D), C-1
    const double com = Phi - Avg + p.gam[q] * J;
    FaceOut o;
    o.cv = s ? W * com : -W * com;                            // [[phi]] = +phi on T-, -phi on T+
    o.cg = -W * 0.5 * J * p.Dqq_h[q];                         // -(nu.{D grad phi}_w, [[u]]): w = 1/2, / h_q
    return o;
}
__device__ __forceinline__ FaceOut flux_boundary(const KParams& p, int q, int s, double W, double uo, double dref)
{
    const double nu = s ? 1.0 : -1.0;                         // outward normal
    const double bn = nu * p.bq[q];
    const double sn = nu * p.Dqq_h[q] * dref;                 // nu . D grad u
    const double Phi = (bn >= 0.0) ? bn * uo : 0.0;           // Phi(u, 0, b_nu)
    FaceOut o;
    o.cv = W * (Phi - sn + p.gam[q] * uo);                    // [[.]] = {.} = v- on the boundary (:282-286)
    o.cg = -W * uo * nu * p.Dqq_h[q];
    return o;
}

template <int N>
__global__ void __launch_bounds__(Cfg<N>::C * N * N)
dg_cell_kernel(const KParams p)
{
    constexpr int C = Cfg<N>::C;
    constexpr int NN = N * N;
    extern __shared__ double smem[];
    static_assert(N == DG_N, "one degree per translation unit");
    const Tab<N>& T = g_tab;

    const int tid = threadIdx.x;
    const int slot = tid / NN;
    const int pi = tid - slot * NN;
    const int a = pi % N, bb = pi / N;

    double* A0 = smem + slot * Smem<N>::PER_CELL;
    double* A1 = A0 + Lay<N>::SLOT;
    double* A2 = A1 + Lay<N>::SLOT;
    double* NT = A2 + Lay<N>::SLOT;

    int64_t task = (int64_t)blockIdx.x * C + slot;
    const bool valid = task < p.ntasks;
    if (!valid) task = p.ntasks - 1;
    int64_t lc[3];
    if (p.task_list) {
        int64_t e = p.task_list[task];
        lc[0] = e % p.nloc[0];
        lc[1] = (e / p.nloc[0]) % p.nloc[1];
        lc[2] = e / (p.nloc[0] * p.nloc[1]);
    } else {
        lc[0] = p.task_lo[0] + task % p.task_cnt[0];
        lc[1] = p.task_lo[1] + (task / p.task_cnt[0]) % p.task_cnt[1];
        lc[2] = p.task_lo[2] + task / (p.task_cnt[0] * p.task_cnt[1]);
    }
    const int64_t n3 = (int64_t)NN * N;
    const int64_t cell = lc[0] + p.nloc[0] * (lc[1] + p.nloc[1] * lc[2]);
    const double* zc = p.z + cell * n3;
    const bool do_int = (p.mask & 2u) != 0, do_bnd = (p.mask & 4u) != 0, do_vol = (p.mask & 1u) != 0;

    // ---------------------------------------------------------------- neighbour traces
    // For face f = 2q + s the neighbour lies at lc[q] + (s ? 1 : -1); its face is x_q = 1 - s.
    // Step A (normal direction first): thread (a, bb) contracts the neighbour's line through
    // tangential modal indices (j_t1 = a, j_t2 = bb) with theta(1-s) and theta'(1-s).
    unsigned nbmask = 0;   // bit f: face f has a neighbour cell (local or on another rank)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int f = 2 * q + s;
            const int64_t g = p.gofs[q] + lc[q] + (s ? 1 : -1);
            int kind = 0;
            if (g >= 0 && g < p.gcells[q]) {
                const int64_t l = lc[q] + (s ? 1 : -1);
                kind = (l >= 0 && l < p.nloc[q]) ? 1 : 2;
            }
            if (kind) nbmask |= 1u << f;
            const bool need = kind != 0 && do_int;
            if (need) {
                const double* zn;
                if (kind == 1) {
                    const int64_t st = (q == 0) ? 1 : (q == 1) ? p.nloc[0] : p.nloc[0] * p.nloc[1];
                    zn = zc + (s ? st : -st) * n3;
                } else {
                    // ghost layer indexed by the two tangential local coordinates
                    const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
                    zn = p.ghost[f] + (lc[t1] + p.nloc[t1] * lc[t2]) * n3;
                }
                const double* thv = s ? T.th0 : T.th1;    // neighbour face is at x_q = 1 - s
                const double* dthv = s ? T.dth0 : T.dth1;
                double su = 0.0, sd = 0.0;
#pragma unroll
                for (int e = 0; e < N; ++e) {
                    int ix, iy, iz;
                    if (q == 0) { ix = e; iy = a; iz = bb; }
                    else if (q == 1) { ix = a; iy = e; iz = bb; }
                    else { ix = a; iy = bb; iz = e; }
                    const double v = __ldg(zn + ix + N * (iy + N * iz));
                    su = fma(thv[e], v, su);
                    sd = fma(dthv[e], v, sd);
                }
                NT[FLay<N>::at(2 * f, a, bb)] = su;
                NT[FLay<N>::at(2 * f + 1, a, bb)] = sd;
            }
        }
    }

    // ---------------------------------------------------------------- (1) evaluate
    double r[N], t[N];
    // x-pencil (y = a, z = bb): coefficients along x from global memory
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = __ldg(zc + e + N * (a + N * bb));
    mv<N>(T.V, r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A0[Lay<N>::at(e, a, bb)] = t[e];
    __syncthreads();

    // neighbour traces, steps B/C: V along t1 then t2 for the 12 arrays (tasks: 12 arrays x N lines)
    {
        constexpr int NTASK = 12 * N;
        for (int task2 = pi; task2 < NTASK; task2 += NN) {
            const int arr = task2 / N, line = task2 % N;
            if (do_int && ((nbmask >> (arr >> 1)) & 1u)) {
#pragma unroll
                for (int e = 0; e < N; ++e) r[e] = NT[FLay<N>::at(arr, e, line)];
                mv<N>(T.V, r, t);
#pragma unroll
                for (int e = 0; e < N; ++e) NT[FLay<N>::at(arr, e, line)] = t[e];
            }
        }
    }

    // y-pencil (x = a, z = bb)
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A0[Lay<N>::at(a, e, bb)];
    mv<N>(T.V, r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A1[Lay<N>::at(a, e, bb)] = t[e];
    __syncthreads();

    {
        constexpr int NTASK = 12 * N;
        for (int task2 = pi; task2 < NTASK; task2 += NN) {
            const int arr = task2 / N, line = task2 % N;
            if (do_int && ((nbmask >> (arr >> 1)) & 1u)) {
#pragma unroll
                for (int e = 0; e < N; ++e) r[e] = NT[FLay<N>::at(arr, line, e)];
                mv<N>(T.V, r, t);
#pragma unroll
                for (int e = 0; e < N; ++e) NT[FLay<N>::at(arr, line, e)] = t[e];
            }
        }
    }

    // z-pencil (x = a, y = bb): u at the Gauss points along z, and d/dz
    double uz[N], dz[N];
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A1[Lay<N>::at(a, bb, e)];
    mv<N>(T.V, r, uz);
    mv<N>(T.Dc, uz, dz);
#pragma unroll
    for (int e = 0; e < N; ++e) A0[Lay<N>::at(a, bb, e)] = uz[e];
    __syncthreads();

    // ---------------------------------------------------------------- faces: own traces + flux
    // wq: tangential quadrature weight product at this thread's face point (a, bb)
    const double wab = T.w[a] * T.w[bb];
    FaceOut fz[2], fx[2], fy[2];
    {
        // z faces at point (x = a, y = bb): traces from uz
        const double W = p.dF[2] * wab;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const double uo = dot<N>(s ? T.L1 : T.L0, uz);
            const double dref = dot<N>(s ? T.LD1 : T.LD0, uz);
            const int f = 4 + s;
            fz[s].cv = 0.0; fz[s].cg = 0.0;
            if ((nbmask >> f) & 1u) {
                if (do_int) {
                    const double un = NT[FLay<N>::at(2 * f, a, bb)];
                    const double sn = p.Dqq_h[2] * NT[FLay<N>::at(2 * f + 1, a, bb)];
                    fz[s] = flux_interior(p, 2, s, W, uo, dref, un, sn);
                }
            } else if (do_bnd) {
                fz[s] = flux_boundary(p, 2, s, W, uo, dref);
            }
        }
    }
    // x-pencil (y = a, z = bb): d/dx and the x-face traces
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A0[Lay<N>::at(e, a, bb)];
    mv<N>(T.Dc, r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A1[Lay<N>::at(e, a, bb)] = t[e];
    {
        const double W = p.dF[0] * wab;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const double uo = dot<N>(s ? T.L1 : T.L0, r);
            const double dref = dot<N>(s ? T.LD1 : T.LD0, r);
            const int f = s;
            fx[s].cv = 0.0; fx[s].cg = 0.0;
            if ((nbmask >> f) & 1u) {
                if (do_int) {
                    const double un = NT[FLay<N>::at(2 * f, a, bb)];
                    const double sn = p.Dqq_h[0] * NT[FLay<N>::at(2 * f + 1, a, bb)];
                    fx[s] = flux_interior(p, 0, s, W, uo, dref, un, sn);
                }
            } else if (do_bnd) {
                fx[s] = flux_boundary(p, 0, s, W, uo, dref);
            }
        }
    }
    // y-pencil (x = a, z = bb): d/dy and the y-face traces
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A0[Lay<N>::at(a, e, bb)];
    mv<N>(T.Dc, r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A2[Lay<N>::at(a, e, bb)] = t[e];
    {
        const double W = p.dF[1] * wab;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const double uo = dot<N>(s ? T.L1 : T.L0, r);
            const double dref = dot<N>(s ? T.LD1 : T.LD0, r);
            const int f = 2 + s;
            fy[s].cv = 0.0; fy[s].cg = 0.0;
            if ((nbmask >> f) & 1u) {
                if (do_int) {
                    const double un = NT[FLay<N>::at(2 * f, a, bb)];
                    const double sn = p.Dqq_h[1] * NT[FLay<N>::at(2 * f + 1, a, bb)];
                    fy[s] = flux_interior(p, 1, s, W, uo, dref, un, sn);
                }
            } else if (do_bnd) {
                fy[s] = flux_boundary(p, 1, s, W, uo, dref);
            }
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- (2) quadrature-point data
    // z-pencil (x = a, y = bb): x^(1..3) as coefficients of the REFERENCE test derivatives,
    // x^(0) = W c u; X = x^(0) + Dc^T x^(3) + z-face lifts stays in registers.
    double X[N];
    {
        const double wxy = p.dT * wab;
        double x1[N], x2[N], x3[N];
#pragma unroll
        for (int e = 0; e < N; ++e) {
            const double gx = A1[Lay<N>::at(a, bb, e)];
            const double gy = A2[Lay<N>::at(a, bb, e)];
            const double gz = dz[e];
            const double u = uz[e];
            const double W = do_vol ? wxy * T.w[e] : 0.0;
            // x^(r) / h_r = W (sum_s D_rs/(h_r h_s) d_s u_hat - b_r/h_r u)     (eq:gauss_points)
            x1[e] = W * (p.Dhat[0] * gx + p.Dhat[1] * gy + p.Dhat[2] * gz - p.kb[0] * u);
            x2[e] = W * (p.Dhat[3] * gx + p.Dhat[4] * gy + p.Dhat[5] * gz - p.kb[1] * u);
            x3[e] = W * (p.Dhat[6] * gx + p.Dhat[7] * gy + p.Dhat[8] * gz - p.kb[2] * u);
            X[e] = W * p.c * u;
        }
#pragma unroll
        for (int e = 0; e < N; ++e) {
            A1[Lay<N>::at(a, bb, e)] = x1[e];
            A2[Lay<N>::at(a, bb, e)] = x2[e];
        }
        mtv<N>(T.Dc, x3, t);
#pragma unroll
        for (int e = 0; e < N; ++e)
            X[e] += t[e] + fz[0].cv * T.L0[e] + fz[0].cg * T.LD0[e] + fz[1].cv * T.L1[e] + fz[1].cg * T.LD1[e];
    }
    __syncthreads();

    // x-pencil: Dc^T x^(1) + x-face lifts (in place in A1)
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A1[Lay<N>::at(e, a, bb)];
    mtv<N>(T.Dc, r, t);
#pragma unroll
    for (int e = 0; e < N; ++e)
        A1[Lay<N>::at(e, a, bb)] = t[e] + fx[0].cv * T.L0[e] + fx[0].cg * T.LD0[e] + fx[1].cv * T.L1[e] + fx[1].cg * T.LD1[e];
    // y-pencil: Dc^T x^(2) + y-face lifts (in place in A2)
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A2[Lay<N>::at(a, e, bb)];
    mtv<N>(T.Dc, r, t);
#pragma unroll
    for (int e = 0; e < N; ++e)
        A2[Lay<N>::at(a, e, bb)] = t[e] + fy[0].cv * T.L0[e] + fy[0].cg * T.LD0[e] + fy[1].cv * T.L1[e] + fy[1].cg * T.LD1[e];
    __syncthreads();

    // ---------------------------------------------------------------- (3) integrate
    // z-pencil: gather, V^T along z
#pragma unroll
    for (int e = 0; e < N; ++e) X[e] += A1[Lay<N>::at(a, bb, e)] + A2[Lay<N>::at(a, bb, e)];
    mtv<N>(T.V, X, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A0[Lay<N>::at(a, bb, e)] = t[e];
    __syncthreads();
    // y-pencil: V^T along y
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A0[Lay<N>::at(a, e, bb)];
    mtv<N>(T.V, r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A1[Lay<N>::at(a, e, bb)] = t[e];
    __syncthreads();
    // x-pencil: V^T along x, then the single store of y (or f - y)
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A1[Lay<N>::at(e, a, bb)];
    mtv<N>(T.V, r, t);
    if (valid) {
        double* yc = p.y + cell * n3 + N * (a + N * bb);
        if (p.f) {
            const double* fc = p.f + cell * n3 + N * (a + N * bb);
#pragma unroll
            for (int e = 0; e < N; ++e) yc[e] = __ldg(fc + e) - t[e];
        } else {
#pragma unroll
            for (int e = 0; e < N; ++e) yc[e] = t[e];
        }
    }
}

}  // namespace dg
