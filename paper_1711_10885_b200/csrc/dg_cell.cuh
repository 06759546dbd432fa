// Fused cell kernel: y = A z for the SIPG/WSIPG operator of arXiv 1711.10885,
// FP64, sm_100a.
//
// Work decomposition: a cell is processed by TPC threads (one warp for n = 7..9, a
// fraction of a warp for small n, two warps for n >= 10); each thread owns P
// "pencils" (lines of n points along one direction) in each of the three roles
// (x-, y- and z-pencil), so one uniform-register load of a 1D matrix entry feeds P
// DFMAs and the cell's phases synchronise with __syncwarp only (no CTA barrier for
// TPC <= 32). The 1D matrices live in __constant__ memory (one copy per use site so
// the compiler reloads per stage instead of hoisting whole matrices into registers).
//
// Per cell (Algorithm 1, reorganised owner-computes):
//   (1) u at the n^3 Gauss points by sum factorization u_q = (V x V x V) z
//       (eq:evalfe; kernel eq:sum_fact_kernel :590-595), each stage
//       by the even-odd decomposition of V (V_{n-1-i,j} = (-1)^j V_ij); the reference
//       gradient by collocation derivatives Dc = G V^{-1} along each pencil (exact on
//       Q_k; Dc is centro-antisymmetric, also applied even-odd)
//   (2) quadrature-point data x^(r) (eq:gauss_points), x^(0) = c u W
//   (3) y = (V^T x V^T x V^T)(x^(0) + sum_r Dc_r^T x^(r) + face lifts)   (eq:evalblf :425-444)
//   (4-10) faces: own traces are 1D extrapolations of u_q along the normal (L_l(s), L'_l(s));
//       neighbour traces are the paper's face sum factorization with the normal direction
//       FIRST: theta(s)/theta'(s) contraction of the neighbour's
//       coefficients, then V along the two tangential directions. Consistency, symmetry,
//       penalty and upwind terms (eq:blf :301-315, Phi :334-341) are evaluated pointwise
//       and lifted with the normal direction LAST into the quadrature-space array before
//       the transposed stages. Each cell writes only its own y block once: no atomics.
#pragma once
#include "dg_internal.h"

namespace dg {

template <int N>
struct EO {                        // even-odd form of a centro-antisymmetric matrix A
    static constexpr int H = N / 2;
    double p[H > 0 ? H : 1][H > 0 ? H : 1];   // (A_ij + A_i,N-1-j) / 2
    double m[H > 0 ? H : 1][H > 0 ? H : 1];   // (A_ij - A_i,N-1-j) / 2
    double col[H > 0 ? H : 1];                // A_iH            (odd N)
    double row[H > 0 ? H : 1];                // A_Hj            (odd N)
};

template <int N>
struct Tab {
    static constexpr int HC = (N + 1) / 2;
    double Vh[10][HC][N];    // V_ij = theta_j(xi_i), rows i < ceil(n/2); one copy per use site
    EO<N> Dc[6];             // collocation derivative Dc_il (row = point, col = value)
    EO<N> DcT[6];            // its transpose
    double w[N];
    double L[6][4][N];       // per use site: L_l(0), L_l(1), L'_l(0), L'_l(1)
    double th0[N], th1[N], dth0[N], dth1[N];
};

#ifndef DG_N
#error "dg_cell.cuh is compiled once per degree with -DDG_N=<k+1>"
#endif
__constant__ Tab<DG_N> g_tab;

// TPC threads per cell, P pencils per thread (TPC * P >= n^2), C cells per CTA.
template <int N> struct Cfg;
template <> struct Cfg<2>  { static constexpr int TPC = 4,  P = 1, C = 32, MINB = 8; };
template <> struct Cfg<3>  { static constexpr int TPC = 8,  P = 2, C = 16, MINB = 8; };
template <> struct Cfg<4>  { static constexpr int TPC = 8,  P = 2, C = 16, MINB = 6; };
template <> struct Cfg<5>  { static constexpr int TPC = 16, P = 2, C = 8,  MINB = 4; };
template <> struct Cfg<6>  { static constexpr int TPC = 16, P = 3, C = 4,  MINB = 8; };
template <> struct Cfg<7>  { static constexpr int TPC = 32, P = 2, C = 1,  MINB = 16; };
template <> struct Cfg<8>  { static constexpr int TPC = 32, P = 2, C = 1,  MINB = 16; };
template <> struct Cfg<9>  { static constexpr int TPC = 32, P = 3, C = 1,  MINB = 12; };
template <> struct Cfg<10> { static constexpr int TPC = 64, P = 2, C = 1,  MINB = 8; };
template <> struct Cfg<11> { static constexpr int TPC = 64, P = 2, C = 1,  MINB = 8; };

// Shared-memory layout of one n^3 cell array: x-, y- and z-pencil accesses of a warp are
// (nearly) bank-conflict free (searched offline; n = 8 uses an XOR swizzle that is conflict
// free for all three access patterns).
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

// Face arrays: 6 faces x 2 quantities x n^2 points, row padded. Slot 2f holds the
// neighbour trace u+, then the lift coefficient cv; slot 2f+1 the neighbour normal
// derivative, then cg.
template <int N> struct FLay {
    static constexpr int RS = N + 1;
    static constexpr int ARR = N * RS + 1;
    static constexpr int SLOT = 12 * ARR;
    __device__ __forceinline__ static int at(int arr, int i1, int i2) { return arr * ARR + i1 + RS * i2; }
};
// n = 8: 64 doubles per array, XOR swizzle conflict free for the three access patterns
// (point (a, b) per lane; lines along i1 and along i2 over 4 consecutive arrays per warp).
template <> struct FLay<8> {
    static constexpr int SLOT = 12 * 64;
    __device__ __forceinline__ static int at(int arr, int i1, int i2)
    {
        return 64 * arr + 8 * (i2 ^ (arr & 1)) + (i1 ^ ((i2 >> 1) | ((arr & 1) << 2)));
    }
};

template <int N>
struct Smem {
    static constexpr int PER_CELL = 3 * Lay<N>::SLOT + FLay<N>::SLOT;
    static constexpr int BYTES = Cfg<N>::C * PER_CELL * 8;
};

// ---------------------------------------------------------------------------------- 1D stages
// t[k][i] = sum_j V_ij r[k][j]  (even-odd: V_{n-1-i,j} = (-1)^j V_ij)
template <int N, int P>
__device__ __forceinline__ void v_fwd(const double (&Vh)[(N + 1) / 2][N], const double (&r)[P][N], double (&t)[P][N])
{
    constexpr int H = N / 2;
#pragma unroll
    for (int i = 0; i < H; ++i) {
        double E[P], O[P];
#pragma unroll
        for (int k = 0; k < P; ++k) { E[k] = 0.0; O[k] = 0.0; }
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
            for (int k = 0; k < P; ++k) {
                if (j & 1) O[k] = fma(Vh[i][j], r[k][j], O[k]);
                else E[k] = fma(Vh[i][j], r[k][j], E[k]);
            }
#pragma unroll
        for (int k = 0; k < P; ++k) {
            t[k][i] = E[k] + O[k];
            t[k][N - 1 - i] = E[k] - O[k];
        }
    }
    if (N & 1) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
            double E = 0.0;
#pragma unroll
            for (int j = 0; j < N; j += 2) E = fma(Vh[H][j], r[k][j], E);
            t[k][H] = E;
        }
    }
}

// t[k][j] = sum_i V_ij r[k][i]
template <int N, int P>
__device__ __forceinline__ void v_bwd(const double (&Vh)[(N + 1) / 2][N], const double (&r)[P][N], double (&t)[P][N])
{
    constexpr int H = N / 2;
    double s[P][H > 0 ? H : 1], d[P][H > 0 ? H : 1];
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int i = 0; i < H; ++i) {
            s[k][i] = r[k][i] + r[k][N - 1 - i];
            d[k][i] = r[k][i] - r[k][N - 1 - i];
        }
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double acc[P];
#pragma unroll
        for (int k = 0; k < P; ++k) acc[k] = ((N & 1) && !(j & 1)) ? Vh[H][j] * r[k][H] : 0.0;
#pragma unroll
        for (int i = 0; i < H; ++i)
#pragma unroll
            for (int k = 0; k < P; ++k) acc[k] = fma(Vh[i][j], (j & 1) ? d[k][i] : s[k][i], acc[k]);
#pragma unroll
        for (int k = 0; k < P; ++k) t[k][j] = acc[k];
    }
}

// t[k] = A r[k] for a centro-antisymmetric A (A_{n-1-i,n-1-j} = -A_ij) in even-odd form
template <int N, int P>
__device__ __forceinline__ void c_apply(const EO<N>& A, const double (&r)[P][N], double (&t)[P][N])
{
    constexpr int H = N / 2;
    double s[P][H > 0 ? H : 1], d[P][H > 0 ? H : 1];
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int j = 0; j < H; ++j) {
            s[k][j] = r[k][j] + r[k][N - 1 - j];
            d[k][j] = r[k][j] - r[k][N - 1 - j];
        }
#pragma unroll
    for (int i = 0; i < H; ++i) {
        double Pp[P], Q[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
            Pp[k] = (N & 1) ? A.col[i] * r[k][H] : 0.0;
            Q[k] = 0.0;
        }
#pragma unroll
        for (int j = 0; j < H; ++j)
#pragma unroll
            for (int k = 0; k < P; ++k) {
                Pp[k] = fma(A.p[i][j], s[k][j], Pp[k]);
                Q[k] = fma(A.m[i][j], d[k][j], Q[k]);
            }
#pragma unroll
        for (int k = 0; k < P; ++k) {
            t[k][i] = Pp[k] + Q[k];
            t[k][N - 1 - i] = Q[k] - Pp[k];
        }
    }
    if (N & 1) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < H; ++j) acc = fma(A.row[j], d[k][j], acc);
            t[k][H] = acc;
        }
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

// ---------------------------------------------------------------------------------- face terms
// Contribution cv * phi_i + cg_phys * d_q phi_i of one face point, returned as
// (cv, cg = cg_phys / h_q, the coefficient of the REFERENCE normal derivative).
// own side s: s = 1 -> face x_q = 1, this cell is T- ; s = 0 -> face x_q = 0, this cell is T+.
struct FaceOut { double cv, cg; };

__device__ __forceinline__ FaceOut flux_interior(const KParams& p, int q, int s, double W, double uo, double dref,
                                                 double un, double sn)
{
    const double so = p.Dqq_h[q] * dref;                      // D_qq du/dx_q (own)
    const double um = s ? uo : un, up = s ? un : uo;
    const double sm = s ? so : sn, sp = s ? sn : so;
    const double bn = p.bq[q];
    const double Phi = (bn >= 0.0) ? bn * um : bn * up;       // upwind flux
    const double J = um - up;                                 // [[u]] = u- - u+
    const double Avg = 0.5 * (sm + sp);                       // nu.{D grad u}_w, w = 1/2 (constant D), C-1
    const double com = Phi - Avg + p.gam[q] * J;
    FaceOut o;
    o.cv = s ? W * com : -W * com;                            // [[phi]] = +phi on T-, -phi on T+
    o.cg = -W * 0.5 * J * p.Dqq_h[q];                         // -(nu.{D grad phi}_w, [[u]])
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

// ---------------------------------------------------------------------------------- kernel
template <int N>
__global__ void __launch_bounds__(Cfg<N>::C * Cfg<N>::TPC, Cfg<N>::MINB)
dg_cell_kernel(const KParams p)
{
    constexpr int TPC = Cfg<N>::TPC, P = Cfg<N>::P, C = Cfg<N>::C;
    constexpr int NN = N * N;
    static_assert(N == DG_N, "one degree per translation unit");
    static_assert(TPC * P >= NN, "pencil slots");
    static_assert(TPC <= 32 || C == 1, "multi-warp cells use CTA barriers: one cell per CTA");
    extern __shared__ double smem[];
    const Tab<N>& T = g_tab;

    const int tid = threadIdx.x;
    const int slot = tid / TPC;
    const int lane = tid - slot * TPC;

    double* A0 = smem + slot * Smem<N>::PER_CELL;
    double* A1 = A0 + Lay<N>::SLOT;
    double* A2 = A1 + Lay<N>::SLOT;
    double* NT = A2 + Lay<N>::SLOT;

    auto csync = [&]() {
        if (TPC <= 32) __syncwarp(); else __syncthreads();
    };

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
        // z fastest within a column; columns in tiles of TX x TY (ragged at the box edge)
        const int64_t nz = p.task_cnt[2], nx = p.task_cnt[0], ny = p.task_cnt[1];
        const int64_t col = task / nz;
        const int64_t TX = p.tile[0], TY = p.tile[1];
        const int64_t ty = col / (TY * nx);
        const int64_t wy = min(TY, ny - ty * TY);
        const int64_t cr = col - ty * TY * nx;
        const int64_t tx = cr / (TX * wy);
        const int64_t wx = min(TX, nx - tx * TX);
        const int64_t ci = cr - tx * TX * wy;
        lc[0] = p.task_lo[0] + tx * TX + ci % wx;
        lc[1] = p.task_lo[1] + ty * TY + ci / wx;
        lc[2] = p.task_lo[2] + (task - col * nz);
    }
    const int64_t n3 = (int64_t)NN * N;
    const int64_t cell = lc[0] + p.nloc[0] * (lc[1] + p.nloc[1] * lc[2]);
    const double* zc = p.z + cell * n3;
    const bool do_int = (p.mask & 2u) != 0, do_bnd = (p.mask & 4u) != 0, do_vol = (p.mask & 1u) != 0;

    // this thread's pencils: pencil index pc = lane + k TPC = a + N bb
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

    // ---------------------------------------------------------------- neighbour traces, step A
    // Face f = 2q + s: the neighbour lies at lc[q] + (s ? 1 : -1) and its face is x_q = 1 - s.
    // Normal direction FIRST: contract the neighbour's line through tangential modal indices
    // (j_t1, j_t2) = (a, bb) with theta(1-s) and theta'(1-s).
    unsigned nbmask = 0;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        const int q = f >> 1, s = f & 1;
        const int64_t g = p.gofs[q] + lc[q] + (s ? 1 : -1);
        if (g >= 0 && g < p.gcells[q]) nbmask |= 1u << f;
    }
    if (do_int) {
        const int64_t lcx = lc[0], lcy = lc[1], lcz = lc[2];
#pragma unroll 1
        for (int q = 0; q < 3; ++q) {
            const int64_t lq = (q == 0) ? lcx : (q == 1) ? lcy : lcz;
            const int64_t nq = (q == 0) ? p.nloc[0] : (q == 1) ? p.nloc[1] : p.nloc[2];
            const int64_t st = (q == 0) ? 1 : (q == 1) ? p.nloc[0] : p.nloc[0] * p.nloc[1];
            const int64_t gi = (q == 0) ? (lcy + p.nloc[1] * lcz) : (q == 1) ? (lcx + p.nloc[0] * lcz)
                                                                              : (lcx + p.nloc[0] * lcy);
            const int se = (q == 0) ? 1 : (q == 1) ? N : NN;
            // both neighbours of this direction: loads of the two faces in flight together
            double rl[P][N], rh[P][N];
            const bool hl = (nbmask >> (2 * q)) & 1u, hh = (nbmask >> (2 * q + 1)) & 1u;
            const double* zl = (lq > 0) ? zc - st * n3 : (hl ? p.ghost[2 * q] + gi * n3 : zc);
            const double* zh = (lq + 1 < nq) ? zc + st * n3 : (hh ? p.ghost[2 * q + 1] + gi * n3 : zc);
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const int base = (q == 0) ? N * pa[k] + NN * pb[k] : (q == 1) ? pa[k] + NN * pb[k] : pa[k] + N * pb[k];
#pragma unroll
                for (int e = 0; e < N; ++e) {
                    rl[k][e] = (act[k] && hl) ? __ldg(zl + base + e * se) : 0.0;
                    rh[k][e] = (act[k] && hh) ? __ldg(zh + base + e * se) : 0.0;
                }
            }
#pragma unroll
            for (int k = 0; k < P; ++k) {
                // low neighbour (face 2q): its face is x_q = 1; high neighbour (2q+1): x_q = 0
                double ul = 0.0, dl = 0.0, uh = 0.0, dh = 0.0;
#pragma unroll
                for (int e = 0; e < N; ++e) {
                    ul = fma(T.th1[e], rl[k][e], ul);
                    dl = fma(T.dth1[e], rl[k][e], dl);
                    uh = fma(T.th0[e], rh[k][e], uh);
                    dh = fma(T.dth0[e], rh[k][e], dh);
                }
                if (act[k]) {
                    if (hl) {
                        NT[FLay<N>::at(4 * q, pa[k], pb[k])] = ul;
                        NT[FLay<N>::at(4 * q + 1, pa[k], pb[k])] = dl;
                    }
                    if (hh) {
                        NT[FLay<N>::at(4 * q + 2, pa[k], pb[k])] = uh;
                        NT[FLay<N>::at(4 * q + 3, pa[k], pb[k])] = dh;
                    }
                }
            }
        }
    }

    // ---------------------------------------------------------------- (1) evaluate
    // x-pencils (y = a, z = bb) straight from global memory, V along x
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const double* src = zc + N * (pa[k] + N * pb[k]);
        if (N % 2 == 0) {
#pragma unroll
            for (int e = 0; e < N; e += 2) {
                const double2 v = act[k] ? __ldg(reinterpret_cast<const double2*>(src + e)) : make_double2(0.0, 0.0);
                r[k][e] = v.x;
                r[k][e + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int e = 0; e < N; ++e) r[k][e] = act[k] ? __ldg(src + e) : 0.0;
        }
    }
    v_fwd<N, P>(T.Vh[0], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A0[Lay<N>::at(e, pa[k], pb[k])] = t[k][e];
    csync();

    // neighbour traces, step B: V along the first tangential index (12 arrays x N lines)
    if (do_int) {
        for (int tk = lane; tk < 12 * N; tk += TPC) {
            const int arr = tk / N, line = tk - arr * N;
            if ((nbmask >> (arr >> 1)) & 1u) {
                double rr[1][N], tt[1][N];
#pragma unroll
                for (int e = 0; e < N; ++e) rr[0][e] = NT[FLay<N>::at(arr, e, line)];
                v_fwd<N, 1>(T.Vh[1], rr, tt);
#pragma unroll
                for (int e = 0; e < N; ++e) NT[FLay<N>::at(arr, e, line)] = tt[0][e];
            }
        }
    }
    // y-pencils (x = a, z = bb): V along y
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(pa[k], e, pb[k])] : 0.0;
    v_fwd<N, P>(T.Vh[2], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A1[Lay<N>::at(pa[k], e, pb[k])] = t[k][e];
    csync();

    // neighbour traces, step C: V along the second tangential index
    if (do_int) {
        for (int tk = lane; tk < 12 * N; tk += TPC) {
            const int arr = tk / N, line = tk - arr * N;
            if ((nbmask >> (arr >> 1)) & 1u) {
                double rr[1][N], tt[1][N];
#pragma unroll
                for (int e = 0; e < N; ++e) rr[0][e] = NT[FLay<N>::at(arr, line, e)];
                v_fwd<N, 1>(T.Vh[3], rr, tt);
#pragma unroll
                for (int e = 0; e < N; ++e) NT[FLay<N>::at(arr, line, e)] = tt[0][e];
            }
        }
    }
    // z-pencils (x = a, y = bb): u at the Gauss points -> A0
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A1[Lay<N>::at(pa[k], pb[k], e)] : 0.0;
    v_fwd<N, P>(T.Vh[4], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A0[Lay<N>::at(pa[k], pb[k], e)] = t[k][e];
    csync();   // step C results visible before the z-face fluxes read NT

    // z faces: traces from this z-pencil of u, fluxes -> NT slots (in place, own point)
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const double W = p.dF[2] * T.w[pa[k]] * T.w[pb[k]];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int f = 4 + s;
            const double uo = dot<N>(T.L[0][s], t[k]);
            const double dref = dot<N>(T.L[0][2 + s], t[k]);
            FaceOut fo = {0.0, 0.0};
            const int i0 = FLay<N>::at(2 * f, pa[k], pb[k]), i1 = FLay<N>::at(2 * f + 1, pa[k], pb[k]);
            if ((nbmask >> f) & 1u) {
                if (do_int) fo = flux_interior(p, 2, s, W, uo, dref, NT[i0], p.Dqq_h[2] * NT[i1]);
            } else if (do_bnd) {
                fo = flux_boundary(p, 2, s, W, uo, dref);
            }
            if (act[k]) { NT[i0] = fo.cv; NT[i1] = fo.cg; }
        }
    }

    // ---------------------------------------------------------------- gradients + x/y faces
    // x-pencils (y = a, z = bb): d/dx_hat -> A1; x-face traces / fluxes
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(e, pa[k], pb[k])] : 0.0;
    c_apply<N, P>(T.Dc[0], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A1[Lay<N>::at(e, pa[k], pb[k])] = t[k][e];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const double W = p.dF[0] * T.w[pa[k]] * T.w[pb[k]];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int f = s;
            const double uo = dot<N>(T.L[1][s], r[k]);
            const double dref = dot<N>(T.L[1][2 + s], r[k]);
            FaceOut fo = {0.0, 0.0};
            const int i0 = FLay<N>::at(2 * f, pa[k], pb[k]), i1 = FLay<N>::at(2 * f + 1, pa[k], pb[k]);
            if ((nbmask >> f) & 1u) {
                if (do_int) fo = flux_interior(p, 0, s, W, uo, dref, NT[i0], p.Dqq_h[0] * NT[i1]);
            } else if (do_bnd) {
                fo = flux_boundary(p, 0, s, W, uo, dref);
            }
            if (act[k]) { NT[i0] = fo.cv; NT[i1] = fo.cg; }
        }
    }
    // y-pencils (x = a, z = bb): d/dy_hat -> A2; y-face traces / fluxes
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(pa[k], e, pb[k])] : 0.0;
    c_apply<N, P>(T.Dc[1], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A2[Lay<N>::at(pa[k], e, pb[k])] = t[k][e];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const double W = p.dF[1] * T.w[pa[k]] * T.w[pb[k]];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int f = 2 + s;
            const double uo = dot<N>(T.L[2][s], r[k]);
            const double dref = dot<N>(T.L[2][2 + s], r[k]);
            FaceOut fo = {0.0, 0.0};
            const int i0 = FLay<N>::at(2 * f, pa[k], pb[k]), i1 = FLay<N>::at(2 * f + 1, pa[k], pb[k]);
            if ((nbmask >> f) & 1u) {
                if (do_int) fo = flux_interior(p, 1, s, W, uo, dref, NT[i0], p.Dqq_h[1] * NT[i1]);
            } else if (do_bnd) {
                fo = flux_boundary(p, 1, s, W, uo, dref);
            }
            if (act[k]) { NT[i0] = fo.cv; NT[i1] = fo.cg; }
        }
    }
    csync();

    // ---------------------------------------------------------------- (2) quadrature-point data
    // z-pencils (x = a, y = bb): u, d/dz_hat; x^(1) -> A1, x^(2) -> A2 (in place);
    // X = x^(0) + Dc^T x^(3) + z-face lifts -> A0 (in place over u)
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(pa[k], pb[k], e)] : 0.0;
    c_apply<N, P>(T.Dc[2], r, t);   // t = d u / dz_hat
    {
        double x3[P][N];
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const double wxy = do_vol ? p.dT * T.w[pa[k]] * T.w[pb[k]] : 0.0;
#pragma unroll
            for (int e = 0; e < N; ++e) {
                const int ie = Lay<N>::at(pa[k], pb[k], e);
                const double gx = act[k] ? A1[ie] : 0.0;
                const double gy = act[k] ? A2[ie] : 0.0;
                const double gz = t[k][e];
                const double u = r[k][e];
                const double W = wxy * T.w[e];
                // x^(r) / h_r = W (sum_s D_rs/(h_r h_s) d_s u_hat - b_r/h_r u)   (eq:gauss_points)
                const double x1 = W * (p.Dhat[0] * gx + p.Dhat[1] * gy + p.Dhat[2] * gz - p.kb[0] * u);
                const double x2 = W * (p.Dhat[3] * gx + p.Dhat[4] * gy + p.Dhat[5] * gz - p.kb[1] * u);
                x3[k][e] = W * (p.Dhat[6] * gx + p.Dhat[7] * gy + p.Dhat[8] * gz - p.kb[2] * u);
                r[k][e] = W * p.c * u;                               // x^(0)
                if (act[k]) { A1[ie] = x1; A2[ie] = x2; }
            }
        }
        c_apply<N, P>(T.DcT[0], x3, t);
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const double cv0 = NT[FLay<N>::at(8, pa[k], pb[k])], cg0 = NT[FLay<N>::at(9, pa[k], pb[k])];
            const double cv1 = NT[FLay<N>::at(10, pa[k], pb[k])], cg1 = NT[FLay<N>::at(11, pa[k], pb[k])];
            if (act[k])
#pragma unroll
                for (int e = 0; e < N; ++e)
                    A0[Lay<N>::at(pa[k], pb[k], e)] = r[k][e] + t[k][e] + cv0 * T.L[3][0][e] + cg0 * T.L[3][2][e] +
                                                      cv1 * T.L[3][1][e] + cg1 * T.L[3][3][e];
        }
    }
    csync();

    // x-pencils: Dc^T x^(1) + x-face lifts (in place in A1)
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A1[Lay<N>::at(e, pa[k], pb[k])] : 0.0;
    c_apply<N, P>(T.DcT[1], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const double cv0 = NT[FLay<N>::at(0, pa[k], pb[k])], cg0 = NT[FLay<N>::at(1, pa[k], pb[k])];
        const double cv1 = NT[FLay<N>::at(2, pa[k], pb[k])], cg1 = NT[FLay<N>::at(3, pa[k], pb[k])];
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e)
                A1[Lay<N>::at(e, pa[k], pb[k])] = t[k][e] + cv0 * T.L[4][0][e] + cg0 * T.L[4][2][e] +
                                                  cv1 * T.L[4][1][e] + cg1 * T.L[4][3][e];
    }
    // y-pencils: Dc^T x^(2) + y-face lifts (in place in A2)
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A2[Lay<N>::at(pa[k], e, pb[k])] : 0.0;
    c_apply<N, P>(T.DcT[2], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const double cv0 = NT[FLay<N>::at(4, pa[k], pb[k])], cg0 = NT[FLay<N>::at(5, pa[k], pb[k])];
        const double cv1 = NT[FLay<N>::at(6, pa[k], pb[k])], cg1 = NT[FLay<N>::at(7, pa[k], pb[k])];
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e)
                A2[Lay<N>::at(pa[k], e, pb[k])] = t[k][e] + cv0 * T.L[5][0][e] + cg0 * T.L[5][2][e] +
                                                  cv1 * T.L[5][1][e] + cg1 * T.L[5][3][e];
    }
    csync();

    // ---------------------------------------------------------------- (3) integrate
    // z-pencils: X = A0 + A1 + A2, V^T along z -> A0
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) {
            const int ie = Lay<N>::at(pa[k], pb[k], e);
            r[k][e] = act[k] ? A0[ie] + A1[ie] + A2[ie] : 0.0;
        }
    v_bwd<N, P>(T.Vh[5], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A0[Lay<N>::at(pa[k], pb[k], e)] = t[k][e];
    csync();
    // y-pencils: V^T along y (in place)
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(pa[k], e, pb[k])] : 0.0;
    v_bwd<N, P>(T.Vh[6], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A0[Lay<N>::at(pa[k], e, pb[k])] = t[k][e];
    csync();
    // x-pencils: V^T along x, then the single store of y (or f - y)
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(e, pa[k], pb[k])] : 0.0;
    v_bwd<N, P>(T.Vh[7], r, t);
    if (valid) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
            if (!act[k]) continue;
            const int64_t off = cell * n3 + N * (pa[k] + N * pb[k]);
            double* yc = p.y + off;
            if (p.f) {
                const double* fc = p.f + off;
#pragma unroll
                for (int e = 0; e < N; ++e) t[k][e] = __ldg(fc + e) - t[k][e];
            }
            if (N % 2 == 0) {
#pragma unroll
                for (int e = 0; e < N; e += 2)
                    __stcs(reinterpret_cast<double2*>(yc + e), make_double2(t[k][e], t[k][e + 1]));
            } else {
#pragma unroll
                for (int e = 0; e < N; ++e) __stcs(yc + e, t[k][e]);
            }
        }
    }
}

}  // namespace dg
