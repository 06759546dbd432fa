// Host-side 1D tables of the CUDA path (product side; independent of oracle/).
//
// Quadrature: m = k+1 point Gauss-Legendre rule on [0,1] (tensor rule),
// nodes by Newton iteration in long double on the shifted Legendre polynomial
// Ptilde_m(x) = P_m(2x-1) using its [0,1] three-term recurrence.
// Basis: orthonormal shifted Legendre theta_j = sqrt(2j+1) Ptilde_j (reading C-2).
//
// Derived tables used by the sum-factorized kernels:
//   V[i][j]  = theta_j(xi_i)                 -- A^(q) of eq:evalfe
//   Dc[i][l] = sum_j theta'_j(xi_i) theta_j(xi_l) w_l
//            = derivative at xi_i of the degree-k interpolant through the Gauss values
//              (exact on Q_k because V^T W V = I, i.e. V^{-1} = V^T W).
//   L{0,1}[l]  = sum_j theta_j(s) theta_j(xi_l) w_l   (Lagrange basis at Gauss points, at s = 0/1)
//   LD{0,1}[l] = sum_j theta'_j(s) theta_j(xi_l) w_l
// These let faces be evaluated / integrated from quadrature-point data along the normal
// direction.
#include "dg_internal.h"

#include <cmath>

namespace dg {

typedef long double ld;

// Ptilde_j(x) and d/dx for j = 0..n-1 (shifted Legendre on [0,1]):
// (j+1) Pt_{j+1} = (2j+1)(2x-1) Pt_j - j Pt_{j-1},  Pt'_{j+1} = Pt'_{j-1} + 2(2j+1) Pt_j
static void shifted_legendre(int n, ld x, ld* P, ld* dP)
{
    P[0] = 1.0L;
    dP[0] = 0.0L;
    if (n > 1) { P[1] = 2.0L * x - 1.0L; dP[1] = 2.0L; }
    for (int j = 1; j + 1 < n; ++j) {
        P[j + 1] = ((2.0L * j + 1.0L) * (2.0L * x - 1.0L) * P[j] - (ld)j * P[j - 1]) / (ld)(j + 1);
        dP[j + 1] = dP[j - 1] + 2.0L * (2.0L * j + 1.0L) * P[j];
    }
}

int build_tables(int k, HostTables* t) { return build_tables_m(k, k + 1, t); }

// m >= k+1 Gauss points (over-integration, NEXT-3): V and G are m x n; the collocation
// derivative Dc and the Lagrange vectors L, L' live on the m points (interpolation with the
// first m basis functions, exact for the degree-k traces and lines).
int build_tables_m(int k, int m, HostTables* t)
{
    if (k < 1 || k > KMAX || m < k + 1 || m > MMAX) return -1;
    const int n = k + 1;
    t->n = n;
    t->m = m;
    ld xi[MMAX], w[MMAX];
    ld P[MMAX + 2], dP[MMAX + 2];
    for (int i = 0; i < m; ++i) {
        // initial guess (ascending): roots of P_m near cos(pi (m - i - 0.25)/(m + 0.5)) mapped to [0,1]
        ld x = 0.5L * (1.0L + cosl(3.14159265358979323846264338327950288L * ((ld)(m - i) - 0.25L) / ((ld)m + 0.5L)));
        for (int it = 0; it < 200; ++it) {
            shifted_legendre(m + 1, x, P, dP);
            ld dx = P[m] / dP[m];
            x -= dx;
            if (fabsl(dx) < 1e-19L) break;
        }
        shifted_legendre(m + 1, x, P, dP);
        xi[i] = x;
        // weight on [0,1]: 1 / (x(1-x) Pt'_m(x)^2)
        w[i] = 1.0L / (x * (1.0L - x) * dP[m] * dP[m]);
    }
    ld th[MMAX][MMAX], dth[MMAX][MMAX];      // theta_j, theta'_j at the m points, j < m
    for (int i = 0; i < m; ++i) {
        shifted_legendre(m, xi[i], P, dP);
        for (int j = 0; j < m; ++j) {
            ld s = sqrtl(2.0L * j + 1.0L);
            th[i][j] = s * P[j];
            dth[i][j] = s * dP[j];
        }
    }
    ld e0[MMAX], e1[MMAX], de0[MMAX], de1[MMAX];
    shifted_legendre(m, 0.0L, P, dP);
    for (int j = 0; j < m; ++j) { ld s = sqrtl(2.0L * j + 1.0L); e0[j] = s * P[j]; de0[j] = s * dP[j]; }
    shifted_legendre(m, 1.0L, P, dP);
    for (int j = 0; j < m; ++j) { ld s = sqrtl(2.0L * j + 1.0L); e1[j] = s * P[j]; de1[j] = s * dP[j]; }

    for (int i = 0; i < m; ++i) {
        t->xi[i] = (double)xi[i];
        t->w[i] = (double)w[i];
        for (int j = 0; j < n; ++j) {
            t->V[i][j] = (double)th[i][j];
            t->G[i][j] = (double)dth[i][j];
        }
        for (int l = 0; l < m; ++l) {
            ld s = 0;
            for (int j = 0; j < m; ++j) s += dth[i][j] * th[l][j];
            t->Dc[i][l] = (double)(s * w[l]);
        }
    }
    for (int l = 0; l < m; ++l) {
        ld a0 = 0, a1 = 0, b0 = 0, b1 = 0;
        for (int j = 0; j < m; ++j) {
            a0 += e0[j] * th[l][j];
            a1 += e1[j] * th[l][j];
            b0 += de0[j] * th[l][j];
            b1 += de1[j] * th[l][j];
        }
        t->L0[l] = (double)(a0 * w[l]);
        t->L1[l] = (double)(a1 * w[l]);
        t->LD0[l] = (double)(b0 * w[l]);
        t->LD1[l] = (double)(b1 * w[l]);
    }
    for (int j = 0; j < n; ++j) {
        t->th0[j] = (double)e0[j];
        t->th1[j] = (double)e1[j];
        t->dth0[j] = (double)de0[j];
        t->dth1[j] = (double)de1[j];
    }
    return 0;
}

}  // namespace dg
