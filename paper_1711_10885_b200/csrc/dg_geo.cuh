// Multilinear-geometry cell kernel: y = A z for the SIPG operator of arXiv 1711.10885 on a
// mesh of Q1-mapped hexahedra (NEXT-3: Problem C's "multilinear geometries", PAPER.md:957-961;
// "x = mu_T(xhat) ... is a d-valued Q_1 finite element function and sum-factorization can be
// used to evaluate its values and derivatives at quadrature points"), with a
// constant (full, symmetric PSD) D, constant b and c, m >= n Gauss points per direction
// (q = 2p, 2p + 4 or Problem C's 3p + 4), FP64.
//
// Per cell (one CTA; one thread per quadrature-space pencil, as dg_vb.cuh):
//   forward: u at the m^3 points by V (m x n) along x, y, z; the reference gradient by the
//     m-point collocation derivative Dc along each direction (exact: u is degree k <= m - 1 on a
//     line);
//   neighbour traces: the normal-first contraction theta(s) . z (or the
//     contraction a neighbour rank sent) then V / G along the two tangential directions: u+ and
//     all three reference derivatives of u+ at the m^2 face points;
//   geometry at every point from the cell's 8 vertices (the Q1 map's Jacobian, J_rs = dx_r/dxi_s,
//     bilinear in the other two coordinates per column), adj(J) = det J J^-1;
//   volume (eq:gauss_points, with the metric terms):
//     x^(r) = W [ (adj D adj^T / det)_rs dhat_s u - (adj b)_r u ],  x^(0) = W c det u;
//   faces (eq:blf): normal N = cof(J) e_q (the cross product of the tangents),
//     nu = N / |N|, dS = |N| dxi; each side's physical gradient with ITS OWN Jacobian; the
//     SIPG + upwind flux per point; the test side c_v phi + c_g nu.D grad phi with
//     nu.D grad phi = (adj D nu / det) . grad_hat phi: the tangential parts become value lifts
//     after a face-level Dc^T stage, the normal part a L'(s) lift, the value part a L(s) lift;
//   backward: y = V^T x V^T x V^T (x^(0) + sum_r Dc_r^T x^(r) + lifts), one store (+ epilogue).
// Each cell writes only its own y block: no atomics.
#pragma once
#include "dg_cell.cuh"

#ifndef DG_M
#error "dg_geo.cuh is compiled once per (n, m) with -DDG_N=<k+1> -DDG_M=<m>"
#endif

namespace dg {
namespace geo {

template <int N, int M>
struct TabG {
    static constexpr int HM = (M + 1) / 2;
    double Vh[HM][N];        // V_ij = theta_j(xi_i), rows i < ceil(m/2) (even-odd over the symmetric rule)
    double G[M][N];          // G_ij = theta'_j(xi_i)
    EO<M> Dc, DcT;           // collocation derivative on the m points and its transpose
    double w[M], xi[M];      // the m-point Gauss rule on [0, 1]
    double L[4][M];          // L_l(0), L_l(1), L'_l(0), L'_l(1) on the m points
    double th0[N], th1[N], dth0[N], dth1[N];
};
__constant__ TabG<DG_N, DG_M> g_tabg;

template <int M> struct GCfg {
    static constexpr int CW = M * M;                              // threads per cell
    static constexpr int C = (M * M <= 32) ? 64 / (M * M) : 1;    // cells per CTA
    static constexpr int TPC = ((C * CW + 31) / 32) * 32;
};
template <int N, int M> struct GLay {                             // one m^3 array (mixed shapes fit)
    static constexpr int SY = M, SZ = M * M + 1;
    static constexpr int SLOT = M * SZ;
    __device__ __forceinline__ static int at(int x, int y, int z) { return x + SY * y + SZ * z; }
};
template <int M> struct GFA {                                     // 6 faces x 4 quantities x m^2 (+1)
    static constexpr int FS = M * M + 1;
    static constexpr int SLOT = 24 * FS;
    __device__ __forceinline__ static int at(int f, int c, int i1, int i2) { return (4 * f + c) * FS + i1 + M * i2; }
};
template <int N, int M> struct GSmem {
    static constexpr int VB = 4 * 4 * 4 * 3;                       // vertex block around the cell
    static constexpr int PER_CELL = 4 * GLay<N, M>::SLOT + GFA<M>::SLOT + VB;
    static constexpr int BYTES = GCfg<M>::C * PER_CELL * 8;
};

// J[r][s] = dx_r / dxi_s of the Q1 map of the cell whose corner (0,0,0) is vertex (ox, oy, oz) of
// the 4 x 4 x 4 block VB[z][y][x][3] (the cell itself at (1, 1, 1), its face neighbours +-1)
__device__ __forceinline__ void jac(const double* VB, int ox, int oy, int oz, double a, double b, double c,
                                    double (&J)[3][3])
{
    auto X = [&](int i, int j, int k, int r) { return VB[(((oz + k) * 4 + (oy + j)) * 4 + (ox + i)) * 3 + r]; };
    const double Ba[2] = {1.0 - a, a}, Bb[2] = {1.0 - b, b}, Bc[2] = {1.0 - c, c};
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        double j0 = 0.0, j1 = 0.0, j2 = 0.0;
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                j0 = fma(Bb[u] * Bc[v], X(1, u, v, r) - X(0, u, v, r), j0);
                j1 = fma(Ba[u] * Bc[v], X(u, 1, v, r) - X(u, 0, v, r), j1);
                j2 = fma(Ba[u] * Bb[v], X(u, v, 1, r) - X(u, v, 0, r), j2);
            }
        J[r][0] = j0;
        J[r][1] = j1;
        J[r][2] = j2;
    }
}
// adj(J) = det J J^-1: row r = (column r+1) x (column r+2) (cyclic); returns det J
__device__ __forceinline__ double adjugate(const double (&J)[3][3], double (&A)[3][3])
{
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const int s = (r + 1) % 3, t = (r + 2) % 3;
        A[r][0] = J[1][s] * J[2][t] - J[2][s] * J[1][t];
        A[r][1] = J[2][s] * J[0][t] - J[0][s] * J[2][t];
        A[r][2] = J[0][s] * J[1][t] - J[1][s] * J[0][t];
    }
    return J[0][0] * A[0][0] + J[1][0] * A[0][1] + J[2][0] * A[0][2];
}

// minimum CTAs per SM (one cell each for m >= 6)
#ifndef DG_GEO_MINB
#define DG_GEO_MINB ((DG_M) <= 13 ? 2 : 1)   // c-k7 (m = 13): 2.8 -> 4.3 GDOF/s; m = 15 spills at 2 (c-k9 2.5 -> 2.2)
#endif
template <int N, int M, bool GH>
__global__ void __launch_bounds__(GCfg<M>::TPC, DG_GEO_MINB)
dg_geo_kernel(const __grid_constant__ KParams p)
{
    constexpr int CW = GCfg<M>::CW, CC = GCfg<M>::C;
    constexpr int NN = N * N, MM = M * M;
    static_assert(N == DG_N && M == DG_M, "one (n, m) per translation unit");
    using LY = GLay<N, M>;
    using FA = GFA<M>;
    extern __shared__ double smem[];
    const TabG<N, M>& T = g_tabg;
    const int slot = threadIdx.x / CW;
    const int lane = (slot < CC) ? threadIdx.x - slot * CW : (1 << 20);   // padding threads: no work
    double* U = smem + (slot < CC ? slot : 0) * GSmem<N, M>::PER_CELL;
    double* DX = U + LY::SLOT;
    double* DY = DX + LY::SLOT;
    double* DZ = DY + LY::SLOT;
    double* F = DZ + LY::SLOT;
    double* VB = F + FA::SLOT;

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
        decode_task(p, task, lc);
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

    // ---- P0: vertex block; x-stage of z (modal x-lines) -> DX(x < m, y, z < n); all neighbour
    //      contractions (normal first) -> face slots c = 0 (value), 1 (normal derivative)
    {
        const int64_t PX = p.nloc[0] + 3, PY = p.nloc[1] + 3;
        for (int t = lane; t < 64 * 3; t += CW) {
            const int r = t % 3, v = t / 3, i = v & 3, j = (v >> 2) & 3, k = v >> 4;
            VB[t] = __ldg(p.vert + ((((int64_t)lc[2] + k) * PY + (lc[1] + j)) * PX + (lc[0] + i)) * 3 + r);
        }
    }
    if (lane < NN) {
        const int ya = lane % N, zb = lane / N;
        double r[N], t[M];
#pragma unroll
        for (int e = 0; e < N; ++e) r[e] = __ldg(zc + N * (ya + N * zb) + e);
        vr_fwd<N, M>(T.Vh, r, t);
#pragma unroll
        for (int e = 0; e < M; ++e) DX[LY::at(e, ya, zb)] = t[e];
        int pa[1] = {ya}, pb[1] = {zb};
        bool act[1] = {true};
#pragma unroll 1
        for (int q = 0; q < 3; ++q) {
            if (!((nbi >> (2 * q)) & 3u)) continue;
            double RL[1][N], RH[1][N];
            const unsigned gm = nb_load<N, 1, GH>(p, zc, n3, q, lc, nbi, pa, pb, act, RL, RH);
            double ul, dl, uh, dh;
            nb_traces<N>(T.th0, T.th1, T.dth0, T.dth1, RL[0], RH[0], gm, ul, dl, uh, dh);
            if ((nbi >> (2 * q)) & 1u) { F[FA::at(2 * q, 0, ya, zb)] = ul; F[FA::at(2 * q, 1, ya, zb)] = dl; }
            if ((nbi >> (2 * q + 1)) & 1u) { F[FA::at(2 * q + 1, 0, ya, zb)] = uh; F[FA::at(2 * q + 1, 1, ya, zb)] = dh; }
        }
    }
    __syncthreads();

    // ---- P1: y-stage DX -> DY(x < m, y < m, z < n); neighbour tangential stage A (along t1, n -> m):
    //      value line -> V (c = 0) and G (c = 2), normal-derivative line -> V (c = 1)
    if (lane < M * N) {
        const int xa = lane % M, zb = lane / M;
        double r[N], t[M];
#pragma unroll
        for (int e = 0; e < N; ++e) r[e] = DX[LY::at(xa, e, zb)];
        vr_fwd<N, M>(T.Vh, r, t);
#pragma unroll
        for (int e = 0; e < M; ++e) DY[LY::at(xa, e, zb)] = t[e];
    }
    for (int t = lane; t < 6 * N; t += CW) {
        const int f = t / N, b = t % N;
        if (!((nbi >> f) & 1u)) continue;
        double ra[N], rd[N], va[M], vd[M], ga[M];
#pragma unroll
        for (int e = 0; e < N; ++e) { ra[e] = F[FA::at(f, 0, e, b)]; rd[e] = F[FA::at(f, 1, e, b)]; }
        vr_fwd<N, M>(T.Vh, ra, va);
        vr_fwd<N, M>(T.Vh, rd, vd);
#pragma unroll
        for (int i = 0; i < M; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) acc = fma(T.G[i][j], ra[j], acc);
            ga[i] = acc;
        }
#pragma unroll
        for (int e = 0; e < M; ++e) {
            F[FA::at(f, 0, e, b)] = va[e];
            F[FA::at(f, 1, e, b)] = vd[e];
            F[FA::at(f, 2, e, b)] = ga[e];
        }
    }
    __syncthreads();

    // ---- P2: z-stage DY -> U (u at the m^3 points); neighbour tangential stage B (along t2):
    //      c = 0: V -> u+, and G -> c = 3 (d/dxi_t2); c = 1: V -> d/dxi_q; c = 2: V -> d/dxi_t1
    if (lane < MM) {
        const int xa = lane % M, yb = lane / M;
        double r[N], t[M];
#pragma unroll
        for (int e = 0; e < N; ++e) r[e] = DY[LY::at(xa, yb, e)];
        vr_fwd<N, M>(T.Vh, r, t);
#pragma unroll
        for (int e = 0; e < M; ++e) U[LY::at(xa, yb, e)] = t[e];
    }
    for (int t = lane; t < 6 * M; t += CW) {
        const int f = t / M, a = t % M;
        if (!((nbi >> f) & 1u)) continue;
        double r0[N], r1[N], r2[N], o[M], g3[M];
#pragma unroll
        for (int e = 0; e < N; ++e) {
            r0[e] = F[FA::at(f, 0, a, e)];
            r1[e] = F[FA::at(f, 1, a, e)];
            r2[e] = F[FA::at(f, 2, a, e)];
        }
#pragma unroll
        for (int i = 0; i < M; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) acc = fma(T.G[i][j], r0[j], acc);
            g3[i] = acc;
        }
        vr_fwd<N, M>(T.Vh, r0, o);
#pragma unroll
        for (int e = 0; e < M; ++e) { F[FA::at(f, 0, a, e)] = o[e]; F[FA::at(f, 3, a, e)] = g3[e]; }
        vr_fwd<N, M>(T.Vh, r1, o);
#pragma unroll
        for (int e = 0; e < M; ++e) F[FA::at(f, 1, a, e)] = o[e];
        vr_fwd<N, M>(T.Vh, r2, o);
#pragma unroll
        for (int e = 0; e < M; ++e) F[FA::at(f, 2, a, e)] = o[e];
    }
    __syncthreads();

    // ---- P3: reference gradient by collocation derivatives: DX, DY, DZ = Dc along x, y, z of U
    if (lane < MM) {
        const int pa = lane % M, pb = lane / M;
#pragma unroll 1
        for (int q = 0; q < 3; ++q) {
            double rr[1][M], gg[1][M];
#pragma unroll
            for (int e = 0; e < M; ++e)
                rr[0][e] = U[q == 0 ? LY::at(e, pa, pb) : (q == 1 ? LY::at(pa, e, pb) : LY::at(pa, pb, e))];
            c_apply<M, 1>(T.Dc, rr, gg);
            double* D = q == 0 ? DX : (q == 1 ? DY : DZ);
#pragma unroll
            for (int e = 0; e < M; ++e)
                D[q == 0 ? LY::at(e, pa, pb) : (q == 1 ? LY::at(pa, e, pb) : LY::at(pa, pb, e))] = gg[0][e];
        }
    }
    __syncthreads();

    // ---- P4: face fluxes at every face point (both sides' traces, each side's own Jacobian);
    //      the face slots are overwritten with the lift coefficients:
    //      c = 0: c_v, 1: c_g w_q (normal), 2: c_g w_t1, 3: c_g w_t2, w = adj(J) D nu / det J
    const double* Dp = p.Dp;
#pragma unroll
    for (int q = 0; q < 3; ++q)                      // (q static: no runtime-indexed local arrays)
    for (int t = lane; t < MM; t += CW) {
        const int a = t % M, b = t / M;
        const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
        const double* Dq[4] = {U, DX, DY, DZ};
        double tr0[4], tr1[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {   // (unrolled: Dq[c] static)
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int l = 0; l < M; ++l) {
                const double v = Dq[c][q == 0 ? LY::at(l, a, b) : (q == 1 ? LY::at(a, l, b) : LY::at(a, b, l))];
                a0 = fma(T.L[0][l], v, a0);
                a1 = fma(T.L[1][l], v, a1);
            }
            tr0[c] = a0;
            tr1[c] = a1;
        }
#pragma unroll 1
        for (int s = 0; s < 2; ++s) {
            const int f = 2 * q + s;
            const bool interior = (nbmask >> f) & 1u;
            if (interior ? !do_int : !do_bnd) {
#pragma unroll
                for (int c = 0; c < 4; ++c) F[FA::at(f, c, a, b)] = 0.0;
                continue;
            }
            // own traces: u and the reference gradient extrapolated along the normal pencil (both
            // faces' in the first pass: each pencil value is read once)
            double tr[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) tr[c] = s ? tr1[c] : tr0[c];
            double xr[3];
            xr[q] = (double)s;
            xr[t1] = T.xi[a];
            xr[t2] = T.xi[b];
            double J[3][3], A[3][3];
            jac(VB, 1, 1, 1, xr[0], xr[1], xr[2], J);
            const double det = adjugate(J, A);
            // N = cof(J) e_q = adj(J)^T e_q = row q of adj(J)  (points to +xi_q)
            const double Nv[3] = {A[q][0], A[q][1], A[q][2]};
            const double area = sqrt(Nv[0] * Nv[0] + Nv[1] * Nv[1] + Nv[2] * Nv[2]);
            const double ia = 1.0 / area;
            const double nu[3] = {Nv[0] * ia, Nv[1] * ia, Nv[2] * ia};
            double Dn[3];
#pragma unroll
            for (int r = 0; r < 3; ++r) Dn[r] = Dp[3 * r] * nu[0] + Dp[3 * r + 1] * nu[1] + Dp[3 * r + 2] * nu[2];
            const double delta = nu[0] * Dn[0] + nu[1] * Dn[1] + nu[2] * Dn[2];
            const double gam = delta * p.sigma;
            // physical gradient grad u = adj^T g / det; its D-normal flux nu.D grad u = (adj Dn) . g / det
            const double idet = 1.0 / det;
            double wv[3];                                   // adj(J) D nu / det: nu.D grad phi = wv . grad_hat phi
#pragma unroll
            for (int r = 0; r < 3; ++r) wv[r] = (A[r][0] * Dn[0] + A[r][1] * Dn[1] + A[r][2] * Dn[2]) * idet;
            const double so = wv[0] * tr[1] + wv[1] * tr[2] + wv[2] * tr[3];
            const double Wf = T.w[a] * T.w[b] * area;
            const double bn = p.bp[0] * nu[0] + p.bp[1] * nu[1] + p.bp[2] * nu[2];
            double cv, cg;
            if (interior) {
                // neighbour: u+, reference gradient (normal, t1, t2 -> by direction), its own Jacobian
                double gn[3];
                gn[q] = F[FA::at(f, 1, a, b)];
                gn[t1] = F[FA::at(f, 2, a, b)];
                gn[t2] = F[FA::at(f, 3, a, b)];
                const double un = F[FA::at(f, 0, a, b)];
                // the neighbour's Jacobian at the common point: its tangential columns are this
                // cell's (the shared face), its normal column the bilinear interpolation of its
                // q-edges at (xi_t1, xi_t2) (a Q1 map's column q does not depend on xi_q)
                double Jn[3][3], An[3][3];
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int c2 = 0; c2 < 3; ++c2) Jn[r][c2] = J[r][c2];
                {
                    int o[3] = {1, 1, 1};
                    o[q] = s ? 2 : 0;
                    auto X = [&](const int (&v)[3], int r) {
                        return VB[(((o[2] + v[2]) * 4 + (o[1] + v[1])) * 4 + (o[0] + v[0])) * 3 + r];
                    };
                    const double B1[2] = {1.0 - T.xi[a], T.xi[a]}, B2[2] = {1.0 - T.xi[b], T.xi[b]};
#pragma unroll
                    for (int r = 0; r < 3; ++r) {
                        double acc = 0.0;
#pragma unroll
                        for (int u = 0; u < 2; ++u)
#pragma unroll
                            for (int v = 0; v < 2; ++v) {
                                int hi[3], lo3[3];
                                hi[q] = 1; lo3[q] = 0;
                                hi[t1] = lo3[t1] = u;
                                hi[t2] = lo3[t2] = v;
                                acc = fma(B1[u] * B2[v], X(hi, r) - X(lo3, r), acc);
                            }
                        Jn[r][q] = acc;
                    }
                }
                const double detn = adjugate(Jn, An);
                double sn = 0.0;
#pragma unroll
                for (int r = 0; r < 3; ++r) sn = fma(An[r][0] * Dn[0] + An[r][1] * Dn[1] + An[r][2] * Dn[2], gn[r], sn);
                sn /= detn;
                const double uo = tr[0];
                const double um = s ? uo : un, up = s ? un : uo;
                const double sm = s ? so : sn, sp = s ? sn : so;
                const double Phi = (bn >= 0.0) ? bn * um : bn * up;     // upwind
                const double Jmp = um - up;
                const double com = Phi - 0.5 * (sm + sp) + gam * Jmp;   // w = 1/2 (one tensor), C-1
                cv = s ? Wf * com : -Wf * com;
                cg = -Wf * 0.5 * Jmp;                                   // times nu.D grad phi (nu to +xi_q)
            } else {
                const double sg = s ? 1.0 : -1.0;                      // outward normal = sg nu
                const double bo = sg * bn;
                const double Phi = (bo >= 0.0) ? bo * tr[0] : 0.0;     // Phi(u, 0, b_nu)
                cv = Wf * (Phi - sg * so + gam * tr[0]);
                cg = -Wf * tr[0] * sg;                                  // -(nu_out.D grad phi) u, as a nu-multiple
            }
            F[FA::at(f, 0, a, b)] = cv;
            F[FA::at(f, 1, a, b)] = cg * wv[q];
            F[FA::at(f, 2, a, b)] = cg * wv[t1];
            F[FA::at(f, 3, a, b)] = cg * wv[t2];
        }
    }
    __syncthreads();

    // ---- P5: volume quadrature data in place (x^(0) -> U, x^(r) -> DX, DY, DZ) on z-pencils;
    //      face-level Dc^T along t1 of the t1 coefficients into the value coefficients
    if (lane < MM) {
        const int pa = lane % M, pb = lane / M;
        const double xa = T.xi[pa], xb = T.xi[pb];
        const double wab = T.w[pa] * T.w[pb];
        // Along this z-pencil (xi_x, xi_y fixed) the Q1 map's Jacobian columns are affine in
        // c = xi_z: J e_x = P0 + c Q0, J e_y = P1 + c Q1, J e_z = C2 (bilinear in (xi_x, xi_y) only);
        // so are the adjugate's rows 0, 1, and row 2 is quadratic. Precomputed once per pencil.
        double P0[3], Q0[3], P1[3], Q1[3], C2[3];
        {
            auto X = [&](int i, int j, int k, int r) { return VB[(((1 + k) * 4 + (1 + j)) * 4 + (1 + i)) * 3 + r]; };
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const double e00 = X(1, 0, 0, r) - X(0, 0, 0, r), e10 = X(1, 1, 0, r) - X(0, 1, 0, r);
                const double e01 = X(1, 0, 1, r) - X(0, 0, 1, r), e11 = X(1, 1, 1, r) - X(0, 1, 1, r);
                P0[r] = (1.0 - xb) * e00 + xb * e10;
                Q0[r] = (1.0 - xb) * (e01 - e00) + xb * (e11 - e10);
                const double f00 = X(0, 1, 0, r) - X(0, 0, 0, r), f10 = X(1, 1, 0, r) - X(1, 0, 0, r);
                const double f01 = X(0, 1, 1, r) - X(0, 0, 1, r), f11 = X(1, 1, 1, r) - X(1, 0, 1, r);
                P1[r] = (1.0 - xa) * f00 + xa * f10;
                Q1[r] = (1.0 - xa) * (f01 - f00) + xa * (f11 - f10);
                const double g00 = X(0, 0, 1, r) - X(0, 0, 0, r), g10 = X(1, 0, 1, r) - X(1, 0, 0, r);
                const double g01 = X(0, 1, 1, r) - X(0, 1, 0, r), g11 = X(1, 1, 1, r) - X(1, 1, 0, r);
                C2[r] = (1.0 - xb) * ((1.0 - xa) * g00 + xa * g10) + xb * ((1.0 - xa) * g01 + xa * g11);
            }
        }
        auto cross = [](const double (&a)[3], const double (&b)[3], double (&o)[3]) {
            o[0] = a[1] * b[2] - a[2] * b[1];
            o[1] = a[2] * b[0] - a[0] * b[2];
            o[2] = a[0] * b[1] - a[1] * b[0];
        };
        double R0a[3], R0b[3], R1a[3], R1b[3], R2a[3], R2b[3], R2c[3], t0[3], t1v[3];
        cross(P1, C2, R0a);                       // row 0 = (J e_y) x (J e_z)
        cross(Q1, C2, R0b);
        cross(C2, P0, R1a);                       // row 1 = (J e_z) x (J e_x)
        cross(C2, Q0, R1b);
        cross(P0, P1, R2a);                       // row 2 = (J e_x) x (J e_y)
        cross(P0, Q1, t0);
        cross(Q0, P1, t1v);
#pragma unroll
        for (int r = 0; r < 3; ++r) R2b[r] = t0[r] + t1v[r];
        cross(Q0, Q1, R2c);
#pragma unroll 1
        for (int e = 0; e < M; ++e) {
            const int ix = LY::at(pa, pb, e);
            const double c = T.xi[e];
            double A[3][3];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                A[0][r] = fma(c, R0b[r], R0a[r]);
                A[1][r] = fma(c, R1b[r], R1a[r]);
                A[2][r] = fma(c, fma(c, R2c[r], R2b[r]), R2a[r]);
            }
            // det J = (J e_x) . row 0
            const double det = fma(c, Q0[0], P0[0]) * A[0][0] + fma(c, Q0[1], P0[1]) * A[0][1] +
                               fma(c, Q0[2], P0[2]) * A[0][2];
            const double W = do_vol ? wab * T.w[e] : 0.0;
            const double g[3] = {DX[ix], DY[ix], DZ[ix]};
            const double u = U[ix];
            // h = adj^T g (= det grad u); x^(r) = W [ adj D h / det - (adj b) u ]_r
            double hv[3], dh[3];
#pragma unroll
            for (int r = 0; r < 3; ++r) hv[r] = A[0][r] * g[0] + A[1][r] * g[1] + A[2][r] * g[2];
#pragma unroll
            for (int r = 0; r < 3; ++r) dh[r] = Dp[3 * r] * hv[0] + Dp[3 * r + 1] * hv[1] + Dp[3 * r + 2] * hv[2];
            const double wd = W / det;
            double x[3];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const double ab = A[r][0] * p.bp[0] + A[r][1] * p.bp[1] + A[r][2] * p.bp[2];
                x[r] = wd * (A[r][0] * dh[0] + A[r][1] * dh[1] + A[r][2] * dh[2]) - W * ab * u;
            }
            DX[ix] = x[0];
            DY[ix] = x[1];
            DZ[ix] = x[2];
            U[ix] = W * p.c * det * u;
        }
    }
    for (int t = lane; t < 6 * M; t += CW) {                  // lines along t1 (i2 = b)
        const int f = t / M, b = t % M;
        double rr[1][M], tt[1][M];
#pragma unroll
        for (int e = 0; e < M; ++e) rr[0][e] = F[FA::at(f, 2, e, b)];
        c_apply<M, 1>(T.DcT, rr, tt);
#pragma unroll
        for (int e = 0; e < M; ++e) F[FA::at(f, 0, e, b)] += tt[0][e];
    }
    __syncthreads();
    for (int t = lane; t < 6 * M; t += CW) {                  // lines along t2 (i1 = a)
        const int f = t / M, a = t % M;
        double rr[1][M], tt[1][M];
#pragma unroll
        for (int e = 0; e < M; ++e) rr[0][e] = F[FA::at(f, 3, a, e)];
        c_apply<M, 1>(T.DcT, rr, tt);
#pragma unroll
        for (int e = 0; e < M; ++e) F[FA::at(f, 0, a, e)] += tt[0][e];
    }
    __syncthreads();

    // ---- P6-P8: roles: x^(0) += Dc_q^T x^(q) + the q-faces' lifts (value L(s), normal L'(s)) along
    //      q-pencils; the z role continues with V^T along z (m -> n) into DX
    const bool actq = lane < MM;
    const int pa = actq ? lane % M : 0, pb = actq ? lane / M : 0;
#pragma unroll 1
    for (int q = 0; q < 3; ++q) {
        if (actq) {
            const double* Xq = q == 0 ? DX : (q == 1 ? DY : DZ);
            double rr[1][M], tt[1][M];
#pragma unroll
            for (int e = 0; e < M; ++e)
                rr[0][e] = Xq[q == 0 ? LY::at(e, pa, pb) : (q == 1 ? LY::at(pa, e, pb) : LY::at(pa, pb, e))];
            c_apply<M, 1>(T.DcT, rr, tt);
            const double cv0 = F[FA::at(2 * q, 0, pa, pb)], cn0 = F[FA::at(2 * q, 1, pa, pb)];
            const double cv1 = F[FA::at(2 * q + 1, 0, pa, pb)], cn1 = F[FA::at(2 * q + 1, 1, pa, pb)];
            double out[M];
#pragma unroll
            for (int e = 0; e < M; ++e) {
                const int ix = q == 0 ? LY::at(e, pa, pb) : (q == 1 ? LY::at(pa, e, pb) : LY::at(pa, pb, e));
                double v = U[ix] + tt[0][e];
                v = fma(cv0, T.L[0][e], fma(cn0, T.L[2][e], v));
                v = fma(cv1, T.L[1][e], fma(cn1, T.L[3][e], v));
                out[e] = v;
            }
            if (q < 2) {
#pragma unroll
                for (int e = 0; e < M; ++e) U[q == 0 ? LY::at(e, pa, pb) : LY::at(pa, e, pb)] = out[e];
            } else {
                double r[N];
                vr_bwd<N, M>(T.Vh, out, r);
#pragma unroll
                for (int e = 0; e < N; ++e) DX[LY::at(pa, pb, e)] = r[e];
            }
        }
        __syncthreads();
    }
    // ---- P9: V^T along y on pencils (x < m, z < n) -> DY(x, y < n, z)
    if (lane < M * N) {
        const int xa = lane % M, zb = lane / M;
        double t[M], r[N];
#pragma unroll
        for (int e = 0; e < M; ++e) t[e] = DX[LY::at(xa, e, zb)];
        vr_bwd<N, M>(T.Vh, t, r);
#pragma unroll
        for (int e = 0; e < N; ++e) DY[LY::at(xa, e, zb)] = r[e];
    }
    __syncthreads();
    // ---- P10: V^T along x on modal pencils (y, z < n); the single store of y (+ epilogue)
    if (lane < NN && valid) {
        const int ya = lane % N, zb = lane / N;
        double t[M], r[N];
#pragma unroll
        for (int e = 0; e < M; ++e) t[e] = DY[LY::at(e, ya, zb)];
        vr_bwd<N, M>(T.Vh, t, r);
        const int64_t off = cell * n3 + N * (ya + N * zb);
        epilogue<N>(p, off, r);
#pragma unroll
        for (int e = 0; e < N; ++e) __stcs(p.y + off + e, r[e]);
    }
}

}  // namespace geo
}  // namespace dg
