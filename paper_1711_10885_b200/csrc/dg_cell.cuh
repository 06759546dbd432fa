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
    // One copy of V / Dc per use site: distinct constant addresses keep the compiler from
    // hoisting a whole 1D matrix into registers across stages (it reloads per stage instead).
    double V[8][N][N];
    double Dc[6][N][N];
    double w[N];
    double L[6][4][N];   // per use site: L_l(0), L_l(1), L'_l(0), L'_l(1)
    double th0[N], th1[N], dth0[N], dth1[N];
};

#ifndef DG_N
#error "dg_cell.cuh is compiled once per degree with -DDG_N=<k+1>"
#endif
// The 1D tables of this translation unit's degree (uploaded by upload_tables).
__constant__ Tab<DG_N> g_tab;

// Cells per CTA for each n (threads = C n^2; 2 CTAs per SM for n = 8).
template <int N> struct Cfg;
template <> struct Cfg<2> { static constexpr int C = 32; static constexpr int MINB = 4; };
template <> struct Cfg<3> { static constexpr int C = 14; static constexpr int MINB = 4; };
template <> struct Cfg<4> { static constexpr int C = 8; static constexpr int MINB = 4; };
template <> struct Cfg<5> { static constexpr int C = 10; static constexpr int MINB = 2; };
template <> struct Cfg<6> { static constexpr int C = 7; static constexpr int MINB = 2; };
template <> struct Cfg<7> { static constexpr int C = 5; static constexpr int MINB = 2; };
template <> struct Cfg<8> { static constexpr int C = 4; static constexpr int MINB = 2; };
template <> struct Cfg<9> { static constexpr int C = 3; static constexpr int MINB = 2; };
template <> struct Cfg<10> { static constexpr int C = 2; static constexpr int MINB = 2; };
template <> struct Cfg<11> { static constexpr int C = 2; static constexpr int MINB = 2; };

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

// Face coefficients of the two faces of one direction at one face point, from the own
// pencil of u at the Gauss points (normal direction q) and the neighbour traces in NT.
template <int N>
__device__ __forceinline__ void face_pair(const KParams& p, const Tab<N>& T, const double* NT, unsigned nbmask,
                                          bool do_int, bool do_bnd, int q, double W, int pt, const double* u,
                                          FaceOut* fo, const double (&Ls)[4][N])
{
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const double uo = dot<N>(Ls[s], u);          // own trace: u(x_q = s)
        const double dref = dot<N>(Ls[2 + s], u);    // own d u / d x_hat_q at x_q = s
        const int f = 2 * q + s;
        fo[s].cv = 0.0;
        fo[s].cg = 0.0;
        if ((nbmask >> f) & 1u) {
            if (do_int) {
                const double un = NT[FLay<N>::ARR * (2 * f) + pt];
                const double sn = p.Dqq_h[q] * NT[FLay<N>::ARR * (2 * f + 1) + pt];
                fo[s] = flux_interior(p, q, s, W, uo, dref, un, sn);
            }
        } else if (do_bnd) {
            fo[s] = flux_boundary(p, q, s, W, uo, dref);
        }
    }
}

// t[e] += lifts of the two faces of one direction along the normal pencil (normal LAST).
template <int N>
__device__ __forceinline__ void add_lift(const double (&Ls)[4][N], const FaceOut* fo, double* t)
{
#pragma unroll
    for (int e = 0; e < N; ++e)
        t[e] += fo[0].cv * Ls[0][e] + fo[0].cg * Ls[2][e] + fo[1].cv * Ls[1][e] + fo[1].cg * Ls[3][e];
}

template <int N>
__global__ void __launch_bounds__(Cfg<N>::C * N * N, Cfg<N>::MINB)
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
        const int64_t e = p.task_list[task];
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

    double r[N], t[N];

    // ---------------------------------------------------------------- own cell: x-pencil stage
    // x-pencil (y = a, z = bb): coefficients along x straight from global memory
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = __ldg(zc + e + N * (a + N * bb));

    // ---------------------------------------------------------------- neighbour traces, step A
    // Face f = 2q + s: the neighbour lies at lc[q] + (s ? 1 : -1) and its face is x_q = 1 - s.
    // Normal direction FIRST: thread (a, bb) contracts the neighbour's line
    // through tangential modal indices (j_t1 = a, j_t2 = bb) with theta(1-s) and theta'(1-s).
    unsigned nbmask = 0;   // bit f: face f has a neighbour cell (local or on another rank)
#pragma unroll 1
    for (int f = 0; f < 6; ++f) {
        const int q = f >> 1, s = f & 1;
        const int64_t g = p.gofs[q] + lc[q] + (s ? 1 : -1);
        if (g < 0 || g >= p.gcells[q]) continue;
        nbmask |= 1u << f;
        if (!do_int) continue;
        const int64_t l = lc[q] + (s ? 1 : -1);
        const double* zn;
        if (l >= 0 && l < p.nloc[q]) {
            const int64_t st = (q == 0) ? 1 : (q == 1) ? p.nloc[0] : p.nloc[0] * p.nloc[1];
            zn = zc + (s ? st : -st) * n3;
        } else {
            // ghost layer (other rank), indexed by the two tangential local coordinates
            const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
            zn = p.ghost[f] + (lc[t1] + p.nloc[t1] * lc[t2]) * n3;
        }
        // element (j_q = e) of the line: offset a*sa + bb*sb + e*se
        const int se = (q == 0) ? 1 : (q == 1) ? N : NN;
        const int base = (q == 0) ? N * a + NN * bb : (q == 1) ? a + NN * bb : a + N * bb;
        const double* thv = s ? T.th0 : T.th1;
        const double* dthv = s ? T.dth0 : T.dth1;
        double su = 0.0, sd = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) {
            const double v = __ldg(zn + base + e * se);
            su = fma(thv[e], v, su);
            sd = fma(dthv[e], v, sd);
        }
        NT[FLay<N>::at(2 * f, a, bb)] = su;
        NT[FLay<N>::at(2 * f + 1, a, bb)] = sd;
    }

    // ---------------------------------------------------------------- (1) evaluate
    mv<N>(T.V[0], r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A0[Lay<N>::at(e, a, bb)] = t[e];
    __syncthreads();

    // neighbour traces, step B: V along the first tangential index (12 arrays x N lines)
    for (int task2 = pi; task2 < 12 * N; task2 += NN) {
        const int arr = task2 / N, line = task2 - arr * N;
        if (do_int && ((nbmask >> (arr >> 1)) & 1u)) {
#pragma unroll
            for (int e = 0; e < N; ++e) r[e] = NT[FLay<N>::at(arr, e, line)];
            mv<N>(T.V[1], r, t);
#pragma unroll
            for (int e = 0; e < N; ++e) NT[FLay<N>::at(arr, e, line)] = t[e];
        }
    }

    // y-pencil (x = a, z = bb)
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A0[Lay<N>::at(a, e, bb)];
    mv<N>(T.V[2], r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A1[Lay<N>::at(a, e, bb)] = t[e];
    __syncthreads();

    // neighbour traces, step C: V along the second tangential index
    for (int task2 = pi; task2 < 12 * N; task2 += NN) {
        const int arr = task2 / N, line = task2 - arr * N;
        if (do_int && ((nbmask >> (arr >> 1)) & 1u)) {
#pragma unroll
            for (int e = 0; e < N; ++e) r[e] = NT[FLay<N>::at(arr, line, e)];
            mv<N>(T.V[3], r, t);
#pragma unroll
            for (int e = 0; e < N; ++e) NT[FLay<N>::at(arr, line, e)] = t[e];
        }
    }

    // z-pencil (x = a, y = bb): u at the Gauss points
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A1[Lay<N>::at(a, bb, e)];
    mv<N>(T.V[4], r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A0[Lay<N>::at(a, bb, e)] = t[e];
    __syncthreads();

    // ---------------------------------------------------------------- faces + gradients
    const double wab = T.w[a] * T.w[bb];          // tangential weights at this face point
    const int pt = a + FLay<N>::RS * bb;          // face point (a, bb) in the NT arrays
    FaceOut fz[2], fx[2], fy[2];
    // z-pencil: z-face traces and fluxes
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A0[Lay<N>::at(a, bb, e)];
    face_pair<N>(p, T, NT, nbmask, do_int, do_bnd, 2, p.dF[2] * wab, pt, r, fz, T.L[0]);
    // x-pencil: d/dx_hat (collocation) and x-face traces / fluxes
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A0[Lay<N>::at(e, a, bb)];
    mv<N>(T.Dc[0], r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A1[Lay<N>::at(e, a, bb)] = t[e];
    face_pair<N>(p, T, NT, nbmask, do_int, do_bnd, 0, p.dF[0] * wab, pt, r, fx, T.L[1]);
    // y-pencil: d/dy_hat and y-face traces / fluxes
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A0[Lay<N>::at(a, e, bb)];
    mv<N>(T.Dc[1], r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A2[Lay<N>::at(a, e, bb)] = t[e];
    face_pair<N>(p, T, NT, nbmask, do_int, do_bnd, 1, p.dF[1] * wab, pt, r, fy, T.L[2]);
    __syncthreads();

    // ---------------------------------------------------------------- (2) quadrature-point data
    // z-pencil (x = a, y = bb): u and d/dz_hat along z; x^(1), x^(2) back to A1, A2 in place,
    // X = x^(0) + Dc^T x^(3) + z-face lifts in registers.
    double X[N];
    {
#pragma unroll
        for (int e = 0; e < N; ++e) r[e] = A0[Lay<N>::at(a, bb, e)];
        double dz[N];
        mv<N>(T.Dc[2], r, dz);
        const double wxy = do_vol ? p.dT * wab : 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) {
            const int ie = Lay<N>::at(a, bb, e);
            const double gx = A1[ie];
            const double gy = A2[ie];
            const double gz = dz[e];
            const double u = r[e];
            const double W = wxy * T.w[e];
            // x^(r) / h_r = W (sum_s D_rs/(h_r h_s) d_s u_hat - b_r/h_r u)   (eq:gauss_points)
            A1[ie] = W * (p.Dhat[0] * gx + p.Dhat[1] * gy + p.Dhat[2] * gz - p.kb[0] * u);
            A2[ie] = W * (p.Dhat[3] * gx + p.Dhat[4] * gy + p.Dhat[5] * gz - p.kb[1] * u);
            t[e] = W * (p.Dhat[6] * gx + p.Dhat[7] * gy + p.Dhat[8] * gz - p.kb[2] * u);
            X[e] = W * p.c * u;
        }
        double s3[N];
        mtv<N>(T.Dc[3], t, s3);
#pragma unroll
        for (int e = 0; e < N; ++e) X[e] += s3[e];
        add_lift<N>(T.L[3], fz, X);
    }
    __syncthreads();

    // x-pencil: Dc^T x^(1) + x-face lifts (in place in A1)
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A1[Lay<N>::at(e, a, bb)];
    mtv<N>(T.Dc[4], r, t);
    add_lift<N>(T.L[4], fx, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A1[Lay<N>::at(e, a, bb)] = t[e];
    // y-pencil: Dc^T x^(2) + y-face lifts (in place in A2)
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A2[Lay<N>::at(a, e, bb)];
    mtv<N>(T.Dc[5], r, t);
    add_lift<N>(T.L[5], fy, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A2[Lay<N>::at(a, e, bb)] = t[e];
    __syncthreads();

    // ---------------------------------------------------------------- (3) integrate
    // z-pencil: gather, V^T along z
#pragma unroll
    for (int e = 0; e < N; ++e) X[e] += A1[Lay<N>::at(a, bb, e)] + A2[Lay<N>::at(a, bb, e)];
    mtv<N>(T.V[5], X, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A0[Lay<N>::at(a, bb, e)] = t[e];
    __syncthreads();
    // y-pencil: V^T along y
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A0[Lay<N>::at(a, e, bb)];
    mtv<N>(T.V[6], r, t);
#pragma unroll
    for (int e = 0; e < N; ++e) A1[Lay<N>::at(a, e, bb)] = t[e];
    __syncthreads();
    // x-pencil: V^T along x, then the single store of y (or f - y)
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = A1[Lay<N>::at(e, a, bb)];
    mtv<N>(T.V[7], r, t);
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
