// Variable-velocity / over-integrated cell kernel: y = A z for the SIPG operator of
// arXiv 1711.10885 with constant diagonal D, a velocity field b(x) evaluated at every
// quadrature point and m >= n Gauss points per direction (NEXT-2/3: the paper's Taylor-Green
// transport run, with q = 2p + 4, i.e. m = k + 3; eq:2 :1093-1100), FP64.
//
// Structure as dg_cell_kernel (Algorithm 1 reorganised owner-computes), with
// rectangular stages: V (m x n, theta_j(xi_i)) maps the n modal values of a line to the m
// Gauss points (eq:evalfe :472-490, sum factorization :573-609), V^T back. The quadrature
// space of a cell is m^3; the three forward stages walk n^2 -> m n -> m^2 pencils and the
// backward stages the reverse. Per direction q on the m-point pencils of u ("role"):
//   g = Dc u (collocation derivative on the m points: exact, u is degree k <= m-1 on a line),
//   own traces u(s), u'(s) by the Lagrange vectors of the m points, the SIPG + upwind flux with
//   the neighbour traces and the pointwise velocity b_q(x) on the face,
//   x^(q) = W (D_qq/h_q^2 g - b_q(x)/h_q u) (eq:gauss_points :455-466), T_q = Dc^T x^(q) + lifts.
// Neighbour traces: normal-first contraction theta(s) . z of the neighbour's modal lines
// (:623-627), then V along both tangential directions (n -> m each).
//
// The velocity field is separable: b_r(x) = amp_r sgn_r f_r0(x_1) f_r1(x_2) f_r2(x_3) with
// f in {1, x, sin x, cos x} (Taylor-Green: cos/sin products; the linear test field: one x),
// so each cell tabulates sin, cos and x at its m Gauss coordinates and 2 face coordinates per
// direction once (3 (m+2) sincos per cell) and every point value is a product of three.
#pragma once
#include "dg_cell.cuh"

#ifndef DG_M
#error "dg_vb.cuh is compiled once per (n, m) with -DDG_N=<k+1> -DDG_M=<m>"
#endif

namespace dg {
namespace vb {

template <int N, int M>
struct TabV {
    static constexpr int HM = (M + 1) / 2;
    double Vh[6][HM][N];     // V_ij = theta_j(xi_i), rows i < ceil(m/2); one copy per use site
    EO<M> Dc[3];             // collocation derivative on the m points
    EO<M> DcT[3];            // its transpose
    double w[M], xi[M];      // the m-point Gauss rule on [0, 1]
    double L[3][4][M];       // L_l(0), L_l(1), L'_l(0), L'_l(1) on the m points
    double th0[N], th1[N], dth0[N], dth1[N];
};
__constant__ TabV<DG_N, DG_M> g_tabv;

// one thread per quadrature-space pencil (CW = m^2 threads per cell); small m packs C cells per
// CTA (all phases are CTA barriers), so the widest phase keeps most threads busy
template <int M> struct VCfg {
    static constexpr int CW = M * M;
    static constexpr int C = (M * M <= 64) ? 128 / (M * M) : 1;
    static constexpr int TPC = ((C * CW + 31) / 32) * 32;
};

template <int N, int M> struct VLay {
    static constexpr int SY = M, SZ = M * M + 1;
    static constexpr int SLOT = M * SZ;
    __device__ __forceinline__ static int at(int x, int y, int z) { return x + SY * y + SZ * z; }
};
// m = 4, 8: the fast kernel's XOR swizzles (dg_cell.cuh Lay / FLay), defined on the whole m^3
// box, so the mixed modal / point shapes of the forward stages index them too (n <= m). With the
// padded linear layout the m = 8 roles' x-pencil reads were 8-way bank conflicts (ncu TG-k5:
// 49 % of the shared-memory wavefronts were conflicts).
template <int N> struct VLay<N, 8> : Lay<8> {};
template <int N> struct VLay<N, 4> : Lay<4> {};
template <int M> struct VFL {                               // 12 face arrays of m x m (+1 pad)
    static constexpr int FS = M * M + 1;
    static constexpr int SLOT = 12 * FS;
    __device__ __forceinline__ static int at(int arr, int i1, int i2) { return arr * FS + i1 + M * i2; }
};
template <> struct VFL<8> : FLaySwz8 {};
template <> struct VFL<4> : FLay<4> {};
#ifndef DG_VB_BULK_NMIN
#define DG_VB_BULK_NMIN 6   // TG k = 5..10 +2.4 / 4.3 / 5.6 / 3.6 / 5.6 / 0.9 %; n = 5 (k = 4) -2.3 %: off
#endif
template <int N, int M> struct VSmem {
    static constexpr int BT = 3 * 4 * (M + 2);               // 1D velocity tables: [dir][fn][point]
    static constexpr int PER_CELL = 2 * VLay<N, M>::SLOT + VFL<M>::SLOT + BT;
    // bulk copies of the own block in (image in B) and of y out (image in A), dg_cell.cuh namespace
    // bulk, where an array holds the shifted n^3 image; + the mbarrier
    static constexpr bool BULK = N >= DG_VB_BULK_NMIN && VLay<N, M>::SLOT >= N * N * N + 1;
    static constexpr int BYTES = VCfg<M>::C * PER_CELL * 8 + (BULK ? 16 : 0);
};

// separable velocity field: function id per (kind, component r, direction d) and sign per (kind, r)
// fn: 0 = x, 1 = sin x, 2 = cos x, 3 = 1
__device__ __forceinline__ int bfn(int kind, int r, int d)
{
    if (kind == 1) {   // Taylor-Green, eq:2: (cos x1 sin(-x2) sin(-x3), 1/2 sin x1 cos(-x2) sin(-x3), 1/2 sin x1 sin(-x2) cos(-x3))
        return (r == d) ? 2 : 1;
    }
    return (d == (r + 1) % 3) ? 0 : 3;   // linear test field b = (x2, x3, x1)
}
__device__ __forceinline__ double bsign(int kind, int r)
{
    // sin(-x) = -sin x, cos(-x) = cos x: r = 0 has two sin(-x) factors, r = 1, 2 one
    return (kind == 1) ? (r == 0 ? 1.0 : -1.0) * (r == 0 ? 1.0 : 0.5) : 1.0;
}

struct Flux { double cv, cg; };

__device__ __forceinline__ Flux vflux_interior(const KParams& p, int q, int s, double W, double bn, double uo,
                                               double dref, double un, double sn)
{
    const double so = p.Dqq_h[q] * dref;
    const double um = s ? uo : un, up = s ? un : uo;
    const double sm = s ? so : sn, sp = s ? sn : so;
    const double Phi = (bn >= 0.0) ? bn * um : bn * up;       // upwind flux with b.nu at the point (:334-341)
    const double J = um - up;
    const double com = Phi - 0.5 * (sm + sp) + p.gam[q] * J;  // w = 1/2 for constant D (C-1)
    Flux o;
    o.cv = s ? W * com : -W * com;
    o.cg = -W * 0.5 * J * p.Dqq_h[q];
    return o;
}
__device__ __forceinline__ Flux vflux_boundary(const KParams& p, int q, int s, double W, double bq, double uo,
                                               double dref)
{
    const double nu = s ? 1.0 : -1.0;
    const double bn = nu * bq;
    const double sn = nu * p.Dqq_h[q] * dref;
    const double Phi = (bn >= 0.0) ? bn * uo : 0.0;           // Phi(u, 0, b_nu) (:309)
    Flux o;
    o.cv = W * (Phi - sn + p.gam[q] * uo);
    o.cg = -W * uo * nu * p.Dqq_h[q];
    return o;
}

template <int N, int M, bool GH>
// minimum CTAs per SM, measured per (n, m) of the Taylor-Green runs (q = 2p + 4): (3, 5) 8
// (TG-k2 13.3 -> 13.6 GDOF/s), (4, 6) 8 (k3 17.5 -> 18.4), (5, 7) 6 (k4 19.2 -> 19.5), (7, 9) 6
// (k6 25.8 -> 27.3); elsewhere the compiler's choice (an explicit minimum of 1 already changed
// the allocation for the worse)
#if defined(DG_VMB)
#define DG_VB_BOUNDS __launch_bounds__(VCfg<M>::TPC, DG_VMB)
#elif (DG_N == 3 && DG_M == 5) || (DG_N == 4 && DG_M == 6)
#define DG_VB_BOUNDS __launch_bounds__(VCfg<M>::TPC, 8)
#elif (DG_N == 5 && DG_M == 7) || (DG_N == 7 && DG_M == 9)
#define DG_VB_BOUNDS __launch_bounds__(VCfg<M>::TPC, 6)
#else
#define DG_VB_BOUNDS __launch_bounds__(VCfg<M>::TPC)
#endif
__global__ void DG_VB_BOUNDS
dg_vb_kernel(const KParams p)
{
    constexpr int TPC = VCfg<M>::CW;                   // stride of the per-cell loops below
    constexpr int CC = VCfg<M>::C;
    constexpr int NN = N * N, MM = M * M;
    static_assert(N == DG_N && M == DG_M, "one (n, m) per translation unit");
    using LY = VLay<N, M>;
    using FL = VFL<M>;
    extern __shared__ double smem[];
    const TabV<N, M>& T = g_tabv;
    const int slot = threadIdx.x / TPC;
    const int lane = (slot < CC) ? threadIdx.x - slot * TPC : (1 << 20);   // padding threads: no work
    double* A = smem + (slot < CC ? slot : 0) * VSmem<N, M>::PER_CELL;
    double* B = A + LY::SLOT;
    double* NT = B + LY::SLOT;
    double* BT = NT + FL::SLOT;                        // [dir][fn][M + 2]

    unsigned task = blockIdx.x * (unsigned)CC + (unsigned)(slot < CC ? slot : 0);
    const bool valid = task < (unsigned)p.ntasks && slot < CC;
    if (task >= (unsigned)p.ntasks) task = (unsigned)p.ntasks - 1u;
    int lc[3];
    if (p.task_list) {
        const unsigned e = (unsigned)p.task_list[task];
        const unsigned nx = (unsigned)p.nloc[0], ny = (unsigned)p.nloc[1];
        lc[0] = (int)(e % nx);
        lc[1] = (int)((e / nx) % ny);
        lc[2] = (int)(e / (nx * ny));
    } else {
        decode_task(p, task, lc);   // the tiled traversal of the fast kernel (L2 reuse of neighbours)
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
    const unsigned nbi = do_int ? nbmask : 0u;
    const int kind = p.bkind;

    // ---- 1D velocity tables of this cell: x, sin x, cos x, 1 at the m Gauss coordinates and x = 0, 1
    //      per direction, copied from the per-rank tables dg_set_velocity computed once
    //      (vel_table_kernel in dg_aux.cu: the same sincos of the same coordinates, so the values
    //      are those the cell would compute; no trigonometric code in this kernel)
    if (kind != 0) {
        for (int i = lane; i < 3 * 4 * (M + 2); i += TPC) {
            const int d = i / (4 * (M + 2)), r = i - d * 4 * (M + 2);
            BT[i] = __ldg(p.vtab + p.vtoff[d] + (int64_t)lc[d] * 4 * (M + 2) + r);
        }
    }
    auto btab = [&](int d, int fn, int e) { return BT[(d * 4 + fn) * (M + 2) + e]; };

    constexpr bool BULK = VSmem<N, M>::BULK;
    double* SB = nullptr;
    bulk::Span bs{};
    if constexpr (BULK) {
        if (p.tma) {
            uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + CC * VSmem<N, M>::PER_CELL);
            bs = bulk::span<N>(zc, B);
            SB = B + bs.sh;
            if (threadIdx.x == 0) tma::mbar_init_n(mbar, CC);
            __syncthreads();
            if (lane == 0) {
                tma::expect_tx(mbar, bs.bytes);
                bulk::load(SB + bs.hd, zc + bs.hd, bs.bytes, mbar);
            }
            tma::wait(mbar, 0);
        }
    }
    double rl[N], rh[N];
    // ---- phase 1: modal x-lines (y, z < n): V along x -> A(x < m, y, z); x-neighbours (normal first)
    if (lane < NN) {
        const int ya = lane % N, zb = lane / N;
        double r[N], t[M];
        if (BULK && SB) {
            const double* src = SB + N * (ya + N * zb);
            if (N % 2 == 0) {
#pragma unroll
                for (int e = 0; e < N; e += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(src + e);
                    r[e] = v.x;
                    r[e + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int e = 0; e < N; ++e) r[e] = src[e];
            }
            if (bs.hd && lane == 0) r[0] = __ldg(zc);
            if (bs.tl && lane == NN - 1) r[N - 1] = __ldg(zc + NN * N - 1);
        } else {
#pragma unroll
            for (int e = 0; e < N; ++e) r[e] = __ldg(zc + N * (ya + N * zb) + e);
        }
        vr_fwd<N, M>(T.Vh[0], r, t);
#pragma unroll
        for (int e = 0; e < M; ++e) A[LY::at(e, ya, zb)] = t[e];
        int pa[1] = {ya}, pb[1] = {zb};
        bool act[1] = {true};
        double RL[1][N], RH[1][N];
        const unsigned gm = nb_load<N, 1, GH>(p, zc, n3, 0, lc, nbi, pa, pb, act, RL, RH);
#pragma unroll
        for (int e = 0; e < N; ++e) { rl[e] = RL[0][e]; rh[e] = RH[0][e]; }
        const bool hl = (nbi >> 0) & 1u, hh = (nbi >> 1) & 1u;
        double ul, dl, uh, dh;
        nb_traces<N>(T.th0, T.th1, T.dth0, T.dth1, rl, rh, gm, ul, dl, uh, dh);
        if (hl) { NT[FL::at(0, ya, zb)] = ul; NT[FL::at(1, ya, zb)] = dl; }
        if (hh) { NT[FL::at(2, ya, zb)] = uh; NT[FL::at(3, ya, zb)] = dh; }
    }
    __syncthreads();

    // neighbour tangential stage (V, n -> m) of the 4 arrays of direction qf along i1 (dim 0,
    // lines i2 < cnt) or i2 (dim 1, lines i1 < cnt)
    auto tangential = [&](int qf, int dim, int cnt) {
        for (int tk = lane; tk < 4 * cnt; tk += TPC) {
            const int arr = 4 * qf + tk / cnt, line = tk % cnt;
            if (!((nbi >> (arr >> 1)) & 1u)) continue;
            double r[N], t[M];
#pragma unroll
            for (int e = 0; e < N; ++e) r[e] = NT[dim ? FL::at(arr, line, e) : FL::at(arr, e, line)];
            vr_fwd<N, M>(T.Vh[1], r, t);
#pragma unroll
            for (int e = 0; e < M; ++e) NT[dim ? FL::at(arr, line, e) : FL::at(arr, e, line)] = t[e];
        }
    };
    // normal-first contraction of q-neighbour modal lines over the n x n tangential modal pencils
    auto contract = [&](int q) {
        if (lane >= NN) return;
        const int pa0 = lane % N, pb0 = lane / N;
        int pa[1] = {pa0}, pb[1] = {pb0};
        bool act[1] = {true};
        double RL[1][N], RH[1][N];
        const unsigned gm = nb_load<N, 1, GH>(p, zc, n3, q, lc, nbi, pa, pb, act, RL, RH);
        const bool hl = (nbi >> (2 * q)) & 1u, hh = (nbi >> (2 * q + 1)) & 1u;
        double ul, dl, uh, dh;
        nb_traces<N>(T.th0, T.th1, T.dth0, T.dth1, RL[0], RH[0], gm, ul, dl, uh, dh);
        if (hl) { NT[FL::at(4 * q, pa0, pb0)] = ul; NT[FL::at(4 * q + 1, pa0, pb0)] = dl; }
        if (hh) { NT[FL::at(4 * q + 2, pa0, pb0)] = uh; NT[FL::at(4 * q + 3, pa0, pb0)] = dh; }
    };

    // ---- phase 2: y-stage on pencils (x < m, z < n) -> B(x, y < m, z); y-neighbours; x-arrays along i1
    if (lane < M * N) {
        const int xa = lane % M, zb = lane / M;
        double r[N], t[M];
#pragma unroll
        for (int e = 0; e < N; ++e) r[e] = A[LY::at(xa, e, zb)];
        vr_fwd<N, M>(T.Vh[2], r, t);
#pragma unroll
        for (int e = 0; e < M; ++e) B[LY::at(xa, e, zb)] = t[e];
    }
    contract(1);
    tangential(0, 0, N);
    __syncthreads();

    // ---- phase 3: z-stage on pencils (x, y < m) -> u = A(x, y, z < m); z-neighbours;
    //      y-arrays along i1, x-arrays along i2
    if (lane < MM) {
        const int xa = lane % M, yb = lane / M;
        double r[N], t[M];
#pragma unroll
        for (int e = 0; e < N; ++e) r[e] = B[LY::at(xa, yb, e)];
        vr_fwd<N, M>(T.Vh[3], r, t);
#pragma unroll
        for (int e = 0; e < M; ++e) A[LY::at(xa, yb, e)] = t[e];
    }
    contract(2);
    tangential(1, 0, N);
    tangential(0, 1, M);
    __syncthreads();

    // ---- roles (phases 4-6) on the quadrature-space pencils (pa along t1, pb along t2)
    const bool actq = lane < MM;
    const int pa = actq ? lane % M : 0, pb = actq ? lane / M : 0;
    double out[M];
    auto role = [&](int q) {
        const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
        double u[M], g[M];
#pragma unroll
        for (int e = 0; e < M; ++e)
            u[e] = A[q == 0 ? LY::at(e, pa, pb) : (q == 1 ? LY::at(pa, e, pb) : LY::at(pa, pb, e))];
        {
            double rr[1][M], gg[1][M];
#pragma unroll
            for (int e = 0; e < M; ++e) rr[0][e] = u[e];
            c_apply<M, 1>(T.Dc[q], rr, gg);
#pragma unroll
            for (int e = 0; e < M; ++e) g[e] = gg[0][e];
        }
        // b_q at this pencil: tangential factor once, the q factor per point
        double btq = 0.0;
        int fq = 3;
        if (kind != 0) {
            btq = p.bamp[q] * bsign(kind, q) * btab(t1, bfn(kind, q, t1), pa) * btab(t2, bfn(kind, q, t2), pb);
            fq = bfn(kind, q, q);
        }
        const double wab = T.w[pa] * T.w[pb];
        const double sw = do_vol ? p.dT * wab : 0.0;
        const double kd = p.Dhat[4 * q];
        double x[M];
#pragma unroll
        for (int e = 0; e < M; ++e) {
            const double bqe = kind ? btq * btab(q, fq, e) : p.bq[q];
            x[e] = sw * T.w[e] * (kd * g[e] - bqe * p.hinv[q] * u[e]);   // x^(q) (eq:gauss_points)
        }
        {
            double rr[1][M], tt[1][M];
#pragma unroll
            for (int e = 0; e < M; ++e) rr[0][e] = x[e];
            c_apply<M, 1>(T.DcT[q], rr, tt);
#pragma unroll
            for (int e = 0; e < M; ++e) out[e] = tt[0][e];
        }
        const double Wf = p.dF[q] * wab;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int f = 2 * q + s;
            const double uo = dot<M>(T.L[q][s], u);
            const double dref = dot<M>(T.L[q][2 + s], u);
            const double bqs = kind ? btq * btab(q, fq, M + s) : p.bq[q];
            Flux fo = {0.0, 0.0};
            if ((nbmask >> f) & 1u) {
                if (do_int) {
                    const double un = NT[FL::at(2 * f, pa, pb)];
                    const double sn = p.Dqq_h[q] * NT[FL::at(2 * f + 1, pa, pb)];
                    fo = vflux_interior(p, q, s, Wf, bqs, uo, dref, un, sn);
                }
            } else if (do_bnd) {
                fo = vflux_boundary(p, q, s, Wf, bqs, uo, dref);
            }
#pragma unroll
            for (int e = 0; e < M; ++e) out[e] = fma(fo.cv, T.L[q][s][e], fma(fo.cg, T.L[q][2 + s][e], out[e]));
        }
        if (q == 2 && do_vol) {
#pragma unroll
            for (int e = 0; e < M; ++e) out[e] = fma(p.dT * wab * T.w[e] * p.c, u[e], out[e]);
        }
    };

    // phase 4: x role -> B; z-arrays along i1, y-arrays along i2
    if (actq) {
        role(0);
#pragma unroll
        for (int e = 0; e < M; ++e) B[LY::at(e, pa, pb)] = out[e];
    }
    tangential(2, 0, N);
    tangential(1, 1, M);
    __syncthreads();
    // phase 5: y role -> B += ; z-arrays along i2
    if (actq) {
        role(1);
#pragma unroll
        for (int e = 0; e < M; ++e) B[LY::at(pa, e, pb)] += out[e];
    }
    tangential(2, 1, M);
    __syncthreads();
    // phase 6: z role (+ reaction) + B, V^T along z (m -> n) -> A(x, y < m, z < n)
    if (actq) {
        role(2);
#pragma unroll
        for (int e = 0; e < M; ++e) out[e] += B[LY::at(pa, pb, e)];
        double r[N];
        vr_bwd<N, M>(T.Vh[4], out, r);
#pragma unroll
        for (int e = 0; e < N; ++e) A[LY::at(pa, pb, e)] = r[e];
    }
    __syncthreads();
    // phase 7: V^T along y on pencils (x < m, z < n) -> B(x, y < n, z)
    if (lane < M * N) {
        const int xa = lane % M, zb = lane / M;
        double t[M], r[N];
#pragma unroll
        for (int e = 0; e < M; ++e) t[e] = A[LY::at(xa, e, zb)];
        vr_bwd<N, M>(T.Vh[5], t, r);
#pragma unroll
        for (int e = 0; e < N; ++e) B[LY::at(xa, e, zb)] = r[e];
    }
    __syncthreads();
    // phase 8: V^T along x on modal pencils (y, z < n); the single store of y (+ epilogue)
    if constexpr (BULK) {
        if (p.tma == 2 && p.epi == 0) {   // through a linear image in A (free) and one bulk store
            double* yc = p.y + cell * n3;
            const bulk::Span ys = bulk::span<N>(yc, A);
            double* S = A + ys.sh;
            if (lane < NN) {
                const int ya = lane % N, zb = lane / N;
                double t[M], r[N];
#pragma unroll
                for (int e = 0; e < M; ++e) t[e] = B[LY::at(e, ya, zb)];
                vr_bwd<N, M>(T.Vh[5], t, r);
                double* dst = S + N * (ya + N * zb);
                if (N % 2 == 0) {
#pragma unroll
                    for (int e = 0; e < N; e += 2) *reinterpret_cast<double2*>(dst + e) = make_double2(r[e], r[e + 1]);
                } else {
#pragma unroll
                    for (int e = 0; e < N; ++e) dst[e] = r[e];
                }
                if (valid && ys.hd && lane == 0) __stcs(yc, r[0]);
                if (valid && ys.tl && lane == NN - 1) __stcs(yc + NN * N - 1, r[N - 1]);
            }
            tma::fence_async();
            __syncthreads();
            if (valid && lane == 0) bulk::store(yc + ys.hd, S + ys.hd, ys.bytes);
            return;
        }
    }
    if (lane < NN && valid) {
        const int ya = lane % N, zb = lane / N;
        double t[M], r[N];
#pragma unroll
        for (int e = 0; e < M; ++e) t[e] = B[LY::at(e, ya, zb)];
        vr_bwd<N, M>(T.Vh[5], t, r);
        const int64_t off = cell * n3 + N * (ya + N * zb);
        epilogue<N>(p, off, r);
#pragma unroll
        for (int e = 0; e < N; ++e) __stcs(p.y + off + e, r[e]);
    }
}

}  // namespace vb
}  // namespace dg
