/*
 * O-1: naive-quadrature oracle for y = A z, the SIPG/WSIPG operator of
 * arXiv 1711.10885, evaluated WITHOUT sum factorization.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * under paper_1711_10885_b200/ and never includes anything from there.
 *
 * What it computes (cell-centric, each cell writes only its own y block):
 *   y_i = a_h(u_z, phi_i)   with a_h the bilinear form eq:blf
 * split into the volume part, interior-face part and boundary-face part
 * (PAPER.md:342-347). Quadrature: tensor Gauss rule with m = k+1 points per
 * direction, exact for every integrand here (constant
 * coefficients, cuboid cells), so the result is the exact bilinear form.
 *
 * Conventions:
 *   reference cell [0,1]^3; theta_j(x) = sqrt(2j+1) P_j(2x-1)   (C-2)
 *   local dof j = jx + n(jy + n jz); cell e = ix + Nx(iy + Ny iz) (C-3)
 *   weighted average {v}_w = w- v- + w+ v+                       (C-1, PAPER.md:271 garbled)
 *   gamma_F = <delta-,delta+> * sigma, delta = nu^T D nu          (C-4)
 *   boundary: [[v]] = {v}_w = v-, gamma = delta*sigma             (C-6)
 *   upwind flux Phi(u-,u+,b_nu) = b_nu u- if b_nu >= 0 else b_nu u+ 
 *   Dirichlet data g = 0 inside A (enters only the RHS)           (C-9)
 *
 * NEXT-1 (the paper's Problem A):
 *   periodic[q] != 0: the two box sides normal to q are glued; the wrap face between
 *     cell N_q-1 (T-) and cell 0 (T+) is an ordinary interior face with nu = +e_q
 *     ("periodic boundaries in the same way as regular processor boundaries", :940-942)
 *   Dcell != NULL: a diffusion tensor per cell (9 doubles row-major, global cell order),
 *     constant inside each cell (Problem A, :945-946); D- and D+ of a face are the
 *     tensors of T- and T+, delta+- = nu^T D+- nu, weights w- = d+/(d-+d+),
 *     w+ = d-/(d-+d+) (:274-281) and gamma = <d-,d+> sigma (:293, :328-333) become live.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t nc[3];     /* cells per direction */
    double lo[3], hi[3];
    int k;             /* polynomial degree (the paper's p) */
    double D[9];       /* diffusion tensor, row-major */
    double b[3];       /* velocity */
    double c;          /* reaction */
    double sigma;      /* D-independent penalty factor (C-4) */
    int periodic[3];   /* per direction: 0 = both sides weak Dirichlet, 1 = periodic (NEXT-1) */
    const double* Dcell; /* NULL: D above everywhere; else per-cell tensors [cell][9] (NEXT-1) */
    int m;             /* Gauss points per direction; 0 -> k+1 (NEXT-3 over-integration) */
    int bkind;         /* 0: constant b above; 1: Taylor-Green; 2: linear test field (NEXT-2) */
    double bamp[3];    /* per-component amplitude of the field (bkind != 0) */
} o1_problem;

/* b(x) at a physical point (bkind != 0): the field times bamp (header). */
static void o1_velocity(const o1_problem* P, const double x[3], double b[3])
{
    if (P->bkind == 1) {
        b[0] = cos(x[0]) * sin(-x[1]) * sin(-x[2]);
        b[1] = 0.5 * sin(x[0]) * cos(-x[1]) * sin(-x[2]);
        b[2] = 0.5 * sin(x[0]) * sin(-x[1]) * cos(-x[2]);
    } else if (P->bkind == 2) {
        b[0] = x[1];
        b[1] = x[2];
        b[2] = x[0];
    } else {
        b[0] = P->b[0]; b[1] = P->b[1]; b[2] = P->b[2];
        return;
    }
    for (int r = 0; r < 3; ++r) b[r] *= P->bamp[r];
}

enum { O1_VOLUME = 1, O1_INTERIOR = 2, O1_BOUNDARY = 4 };

#define O1_NMAX 16

/* Legendre P_0..P_{n-1} and derivatives at t in [-1,1] by the Bonnet
 * three-term recurrence (n+1) P_{n+1} = (2n+1) t P_n - n P_{n-1}, and
 * P'_{n+1} = (n+1) P_n + t P'_n. */
static void o1_legendre(int n, double t, double* P, double* dP)
{
    P[0] = 1.0; dP[0] = 0.0;
    if (n > 1) { P[1] = t; dP[1] = 1.0; }
    for (int j = 1; j + 1 < n; ++j) {
        P[j + 1] = ((2.0 * j + 1.0) * t * P[j] - j * P[j - 1]) / (j + 1.0);
        dP[j + 1] = (j + 1.0) * P[j] + t * dP[j];
    }
}

/* Orthonormal shifted Legendre basis on [0,1] (C-2):
 * theta_j(x) = sqrt(2j+1) P_j(2x-1), theta'_j(x) = 2 sqrt(2j+1) P'_j(2x-1). */
static void o1_theta(int n, double x, double* th, double* dth)
{
    double P[O1_NMAX + 1], dP[O1_NMAX + 1];
    o1_legendre(n, 2.0 * x - 1.0, P, dP);
    for (int j = 0; j < n; ++j) {
        double s = sqrt(2.0 * j + 1.0);
        th[j] = s * P[j];
        dth[j] = 2.0 * s * dP[j];
    }
}

/* m-point Gauss-Legendre rule on [0,1] by Newton iteration on P_m
 * (PAPER.md:404-416 uses a tensor Gauss rule; SPEC.md:96-98 the recipe). */
static void o1_gauss(int m, double* xi, double* w)
{
    for (int i = 0; i < m; ++i) {
        double t = cos(M_PI * (i + 0.75) / (m + 0.5));
        double P[O1_NMAX + 2], dP[O1_NMAX + 2];
        for (int it = 0; it < 100; ++it) {
            o1_legendre(m + 1, t, P, dP);
            double dt = P[m] / dP[m];
            t -= dt;
            if (fabs(dt) < 1e-16) break;
        }
        o1_legendre(m + 1, t, P, dP);
        /* map [-1,1] -> [0,1]: x = (1+t)/2, weight 2/((1-t^2)P'_m^2) halved */
        xi[i] = 0.5 * (1.0 + t);
        w[i] = 1.0 / ((1.0 - t * t) * dP[m] * dP[m]);
    }
    /* sort ascending */
    for (int a = 0; a < m; ++a)
        for (int b2 = a + 1; b2 < m; ++b2)
            if (xi[b2] < xi[a]) {
                double tx = xi[a]; xi[a] = xi[b2]; xi[b2] = tx;
                double tw = w[a]; w[a] = w[b2]; w[b2] = tw;
            }
}

/* Exported so tests can pin the oracle's tables against closed forms. */
int o1_tables(int k, double* xi, double* w, double* theta_at, double* dtheta_at,
              double* theta0, double* theta1, double* dtheta0, double* dtheta1)
{
    int n = k + 1, m = k + 1;
    if (k < 0 || n > O1_NMAX) return -1;
    o1_gauss(m, xi, w);
    for (int i = 0; i < m; ++i) o1_theta(n, xi[i], theta_at + i * n, dtheta_at + i * n);
    o1_theta(n, 0.0, theta0, dtheta0);
    o1_theta(n, 1.0, theta1, dtheta1);
    return 0;
}

/* Exported so tests can pin the velocity field O-1 evaluates at its quadrature points
 * (o1_velocity above; eq:2) against hand values and div b = 0.
 * x: npts points (x1, x2, x3) interleaved; b: npts velocities, same layout. */
int o1_velocity_at(int bkind, const double* bamp, const double* x, double* b, int64_t npts)
{
    if (bkind < 0 || bkind > 2 || npts < 0) return -1;
    o1_problem P;
    memset(&P, 0, sizeof(P));
    P.bkind = bkind;
    for (int r = 0; r < 3; ++r) P.bamp[r] = bamp ? bamp[r] : 1.0;
    for (int64_t i = 0; i < npts; ++i) o1_velocity(&P, x + 3 * i, b + 3 * i);
    return 0;
}

typedef struct {
    int n, m;
    double h[3];
    double xi[O1_NMAX], w[O1_NMAX];
    double th[O1_NMAX][O1_NMAX], dth[O1_NMAX][O1_NMAX];  /* [point][basis] */
    double th_end[2][O1_NMAX], dth_end[2][O1_NMAX];       /* [x=0 / x=1][basis] */
} o1_tab;

/* Value and PHYSICAL gradient of the FE function of one cell at a reference
 * point given per direction either as a Gauss index (>=0) or an endpoint
 * (-1 -> x=0, -2 -> x=1). Direct sum over all n^3 basis functions
 * (eq:evalfe, without factorization). */
static void o1_eval(const o1_tab* T, const double* zc, const int pidx[3], double* u, double g[3])
{
    int n = T->n;
    const double *v[3], *d[3];
    for (int q = 0; q < 3; ++q) {
        if (pidx[q] >= 0) { v[q] = T->th[pidx[q]]; d[q] = T->dth[pidx[q]]; }
        else { v[q] = T->th_end[-pidx[q] - 1]; d[q] = T->dth_end[-pidx[q] - 1]; }
    }
    double su = 0, s0 = 0, s1 = 0, s2 = 0;
    for (int jz = 0; jz < n; ++jz)
        for (int jy = 0; jy < n; ++jy)
            for (int jx = 0; jx < n; ++jx) {
                double zj = zc[jx + n * (jy + n * jz)];
                su += zj * v[0][jx] * v[1][jy] * v[2][jz];
                s0 += zj * d[0][jx] * v[1][jy] * v[2][jz];
                s1 += zj * v[0][jx] * d[1][jy] * v[2][jz];
                s2 += zj * v[0][jx] * v[1][jy] * d[2][jz];
            }
    *u = su;
    g[0] = s0 / T->h[0];
    g[1] = s1 / T->h[1];
    g[2] = s2 / T->h[2];
}

/* y_i += cv * phi_i(p) + sum_r cg[r] * d_r phi_i(p) for every local test i. */
static void o1_accum(const o1_tab* T, double* yc, const int pidx[3], double cv, const double cg[3])
{
    int n = T->n;
    const double *v[3], *d[3];
    for (int q = 0; q < 3; ++q) {
        if (pidx[q] >= 0) { v[q] = T->th[pidx[q]]; d[q] = T->dth[pidx[q]]; }
        else { v[q] = T->th_end[-pidx[q] - 1]; d[q] = T->dth_end[-pidx[q] - 1]; }
    }
    for (int jz = 0; jz < n; ++jz)
        for (int jy = 0; jy < n; ++jy)
            for (int jx = 0; jx < n; ++jx) {
                double phi = v[0][jx] * v[1][jy] * v[2][jz];
                double d0 = d[0][jx] * v[1][jy] * v[2][jz] / T->h[0];
                double d1 = v[0][jx] * d[1][jy] * v[2][jz] / T->h[1];
                double d2 = v[0][jx] * v[1][jy] * d[2][jz] / T->h[2];
                yc[jx + n * (jy + n * jz)] += cv * phi + cg[0] * d0 + cg[1] * d1 + cg[2] * d2;
            }
}

static double o1_harmonic(double a, double b)
{
    return (a + b == 0.0) ? 0.0 : 2.0 * a * b / (a + b);   /* PAPER.md:293, C-5 */
}

/* Compute the y block of one cell (global cell index e) into yc[n^3]. */
static void o1_cell(const o1_problem* P, const o1_tab* T, const double* z, int64_t e,
                    unsigned mask, double* yc)
{
    int n = T->n, m = T->m;
    int64_t n3 = (int64_t)n * n * n;
    int64_t ic[3];
    ic[0] = e % P->nc[0];
    ic[1] = (e / P->nc[0]) % P->nc[1];
    ic[2] = e / (P->nc[0] * P->nc[1]);
    int64_t stride[3] = {1, P->nc[0], P->nc[0] * P->nc[1]};
    const double* zc = z + e * n3;
    const double* D = P->Dcell ? P->Dcell + 9 * e : P->D;   /* this cell's tensor */
    double dT = T->h[0] * T->h[1] * T->h[2];
    memset(yc, 0, sizeof(double) * n3);

    /* ---- volume term: ((D grad u - b u), grad v)_T + (c u, v)_T */
    if (mask & O1_VOLUME) {
        for (int a3 = 0; a3 < m; ++a3)
            for (int a2 = 0; a2 < m; ++a2)
                for (int a1 = 0; a1 < m; ++a1) {
                    int p[3] = {a1, a2, a3};
                    double u, g[3];
                    o1_eval(T, zc, p, &u, g);
                    double W = dT * T->w[a1] * T->w[a2] * T->w[a3];
                    double xp[3], bp[3];
                    for (int r = 0; r < 3; ++r) xp[r] = P->lo[r] + ((double)ic[r] + T->xi[p[r]]) * T->h[r];
                    o1_velocity(P, xp, bp);
                    double F[3];
                    for (int r = 0; r < 3; ++r)
                        F[r] = W * (D[3 * r + 0] * g[0] + D[3 * r + 1] * g[1] + D[3 * r + 2] * g[2] - bp[r] * u);
                    o1_accum(T, yc, p, W * P->c * u, F);
                }
    }

    /* ---- faces: 6 per cell; q = normal direction, s = 0 (low, x_q=0) or 1 (high) */
    for (int q = 0; q < 3; ++q) {
        int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
        double dF = dT / T->h[q];
        double Dqq = D[3 * q + q];
        for (int s = 0; s < 2; ++s) {
            int64_t nb_i = ic[q] + (s ? 1 : -1);
            int interior = (nb_i >= 0 && nb_i < P->nc[q]);
            if (!interior && P->periodic[q]) {                  /* wrap: glued box sides */
                nb_i = (nb_i < 0) ? P->nc[q] - 1 : 0;
                interior = 1;
            }
            if (interior && !(mask & O1_INTERIOR)) continue;
            if (!interior && !(mask & O1_BOUNDARY)) continue;
            int64_t enb = e + (nb_i - ic[q]) * stride[q];       /* neighbour cell id */
            const double* zn = interior ? z + enb * n3 : NULL;
            const double* Dn = (interior && P->Dcell) ? P->Dcell + 9 * enb : D;
            const double* Dm_ = s ? D : Dn;                     /* tensor of T- */
            const double* Dp_ = s ? Dn : D;                     /* tensor of T+ */
            for (int b2 = 0; b2 < m; ++b2)
                for (int b1 = 0; b1 < m; ++b1) {
                    int pown[3], pnb[3];
                    pown[t1] = b1; pown[t2] = b2; pown[q] = s ? -2 : -1;       /* own face x_q = s */
                    pnb[t1] = b1;  pnb[t2] = b2;  pnb[q] = s ? -1 : -2;        /* neighbour's x_q = 1-s */
                    double W = dF * T->w[b1] * T->w[b2];
                    double u, g[3];
                    o1_eval(T, zc, pown, &u, g);
                    double xf[3], bf[3];     /* the face point (own cell's coordinates) and b there */
                    xf[q] = P->lo[q] + ((double)ic[q] + (double)s) * T->h[q];
                    xf[t1] = P->lo[t1] + ((double)ic[t1] + T->xi[b1]) * T->h[t1];
                    xf[t2] = P->lo[t2] + ((double)ic[t2] + T->xi[b2]) * T->h[t2];
                    o1_velocity(P, xf, bf);
                    if (interior) {
                        /* nu = +e_q oriented from T- (low cell) to T+ (high cell) */
                        double un, gn[3];
                        o1_eval(T, zn, pnb, &un, gn);
                        double um = s ? u : un, up = s ? un : u;
                        const double* gm = s ? g : gn;
                        const double* gp = s ? gn : g;
                        double sm = Dm_[3 * q + 0] * gm[0] + Dm_[3 * q + 1] * gm[1] + Dm_[3 * q + 2] * gm[2];
                        double sp = Dp_[3 * q + 0] * gp[0] + Dp_[3 * q + 1] * gp[1] + Dp_[3 * q + 2] * gp[2];
                        double dm = Dm_[3 * q + q], dp = Dp_[3 * q + q];  /* delta = nu^T D nu */
                        double wm, wp;
                        if (dm + dp == 0.0) { wm = 0.5; wp = 0.5; }  /* C-5 */
                        else { wm = dp / (dm + dp); wp = dm / (dm + dp); }
                        double gam = o1_harmonic(dm, dp) * P->sigma;
                        double bn = bf[q];
                        double Phi = (bn >= 0.0) ? bn * um : bn * up;
                        double J = um - up;
                        double Avg = wm * sm + wp * sp;          /* C-1: "+" reading */
                        double common = Phi - Avg + gam * J;
                        /* test on T-: [[v]] = v, {D grad v}_w = w- D grad v;
                           test on T+: [[v]] = -v, {D grad v}_w = w+ D grad v   (eq:blf) */
                        double sign = s ? 1.0 : -1.0;
                        double wself = s ? wm : wp;
                        double cv = W * sign * common;
                        double cg[3];
                        for (int r = 0; r < 3; ++r) cg[r] = -W * wself * J * D[3 * q + r];
                        o1_accum(T, yc, pown, cv, cg);
                    } else {
                        /* Dirichlet boundary face, outward normal nu = (2s-1) e_q */
                        double nu = s ? 1.0 : -1.0;
                        double bn = nu * bf[q];
                        double sn = nu * (D[3 * q + 0] * g[0] + D[3 * q + 1] * g[1] + D[3 * q + 2] * g[2]);
                        double Phi = (bn >= 0.0) ? bn * u : 0.0;   /* Phi(u, 0, b_nu) */
                        double gam = Dqq * P->sigma;               /* C-6 */
                        double cv = W * (Phi - sn + gam * u);
                        double cg[3];
                        for (int r = 0; r < 3; ++r) cg[r] = -W * u * nu * D[3 * q + r];
                        o1_accum(T, yc, pown, cv, cg);
                    }
                }
        }
    }
}

static void o1_setup_tab(const o1_problem* P, o1_tab* T)
{
    int n = P->k + 1;
    int m = P->m > 0 ? P->m : n;
    T->n = n;
    T->m = m;
    for (int q = 0; q < 3; ++q) T->h[q] = (P->hi[q] - P->lo[q]) / (double)P->nc[q];
    o1_gauss(m, T->xi, T->w);
    for (int i = 0; i < m; ++i) o1_theta(n, T->xi[i], T->th[i], T->dth[i]);
    o1_theta(n, 0.0, T->th_end[0], T->dth_end[0]);
    o1_theta(n, 1.0, T->th_end[1], T->dth_end[1]);
}

/*
 * y = A z restricted to the cells in `cells` (all cells if cells == NULL).
 * compact != 0: the block of cells[i] goes to y + i*n^3; else to y + cells[i]*n^3.
 * nthreads <= 0: OpenMP default. Returns the number of threads used, <0 on error.
 */
int o1_apply(const o1_problem* P, const double* z, double* y, unsigned mask,
             const int64_t* cells, int64_t ncell_list, int compact, int nthreads)
{
    if (P->k < 0 || P->k + 1 > O1_NMAX || P->m > O1_NMAX || (P->m > 0 && P->m < P->k + 1)) return -1;
    o1_tab T;
    o1_setup_tab(P, &T);
    int64_t n3 = (int64_t)T.n * T.n * T.n;
    int64_t total = P->nc[0] * P->nc[1] * P->nc[2];
    int64_t cnt = cells ? ncell_list : total;
    int used = 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
    {
#pragma omp single
        used = omp_get_num_threads();
#pragma omp for schedule(dynamic, 4)
        for (int64_t i = 0; i < cnt; ++i) {
            int64_t e = cells ? cells[i] : i;
            o1_cell(P, &T, z, e, mask, y + (compact ? i : e) * n3);
        }
    }
#else
    (void)nthreads;
    for (int64_t i = 0; i < cnt; ++i) {
        int64_t e = cells ? cells[i] : i;
        o1_cell(P, &T, z, e, mask, y + (compact ? i : e) * n3);
    }
#endif
    return used;
}
