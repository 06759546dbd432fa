"""Right-hand side l_h, L2 projection and the upwind energy functional (numpy).
TEST INFRASTRUCTURE ONLY.

- l_h(v) = sum_T (f, v)_T - sum_{F in F^N} (j, v)_F - sum_{F in F^D} (Phi(0, g, nu.b), v)_F
           - sum_{F in F^D} (nu.(D grad v), g)_F + sum_{F in F^D} gamma_F (g, v)_F
  (Neumann part absent: all faces Dirichlet, reading C-10;
  gamma_F on the boundary = nu^T D nu * sigma, reading C-6).
- Polynomial consistency: for u* in Q_k the SIPG form is consistent, so with
  z* the cell-wise L2 projection of u* and f = -div(D grad u*) + b.grad u* + c u*,
  g = u*|boundary:   A z* = F  (up to rounding). Pins reading C-1 (sign of the
  weighted average) and every sign of eq:blf.
- Upwind energy identity (D = 0, c = 0, constant b, div b = 0):
  z^T A z = 1/2 sum_{F interior} |b_nu| int_F [[u]]^2 + 1/2 sum_{F boundary} |b_nu| int_F u^2
  (follows from the upwind flux definition PAPER.md:334-341 by integrating
  -(b u, grad u)_T = -1/2 int_{dT} b.nu u^2 cell by cell).
"""
import numpy as np
from numpy.polynomial import legendre as npleg

from .tables import gauss01, theta


class PolyField:
    """u*(x) = sum_{a,b,c<=k} alpha_abc P_a(X) P_b(Y) P_c(Z), X = affine map of the box to [-1,1]."""

    def __init__(self, k, lo, hi, seed):
        rng = np.random.default_rng(seed)
        self.alpha = rng.uniform(-1.0, 1.0, size=(k + 1, k + 1, k + 1))   # [a][b][c]
        self.lo = np.asarray(lo, float)
        self.hi = np.asarray(hi, float)
        self.k = k

    def _tabs(self, q, x, der):
        """[len(x), k+1] table of d^der/dx^der P_a(X(x))."""
        L = self.hi[q] - self.lo[q]
        X = 2.0 * (np.asarray(x) - self.lo[q]) / L - 1.0
        out = np.empty((np.size(x), self.k + 1))
        for a in range(self.k + 1):
            c = np.zeros(a + 1)
            c[a] = 1.0
            if der:
                c = npleg.legder(c, der) * (2.0 / L) ** der
            out[:, a] = npleg.legval(X, c) if c.size else 0.0
        return out

    def eval(self, x, y, z, d=(0, 0, 0)):
        """Derivative d of u* at the tensor grid x (fastest) x y x z; returns [z, y, x]."""
        tx, ty, tz = self._tabs(0, x, d[0]), self._tabs(1, y, d[1]), self._tabs(2, z, d[2])
        return np.einsum("abc,ia,jb,kc->kji", self.alpha, tx, ty, tz)


def _cell_points(lo, h, ic, xi):
    return [lo[q] + (ic[q] + xi) * h[q] for q in range(3)]


class KinkedField:
    """u*(x) continuous and piecewise linear in x with a kink at every cell interface
    x = lo + i h_x; on layer i the slope is F / d_i, so the normal flux d_i du/dx = F is
    continuous across every face although D jumps (NEXT-1: discontinuous per-cell D).
    u* lies in Q_1 on each cell, so it is reproduced exactly for every k >= 1."""

    def __init__(self, lo, hx, d_layers, flux, u0):
        self.lo, self.hx = float(lo), float(hx)
        self.slope = flux / np.asarray(d_layers, float)
        self.u_at = u0 + np.concatenate([[0.0], np.cumsum(self.slope * hx)])   # u at the layer starts

    def eval(self, x, y, z, d=(0, 0, 0)):
        x = np.asarray(x, float)
        i = np.clip(np.floor((x - self.lo) / self.hx + 1e-12).astype(int), 0, len(self.slope) - 1)
        if d[1] or d[2] or d[0] > 1:
            vx = np.zeros_like(x)
        elif d[0] == 1:
            vx = self.slope[i]
        else:
            vx = self.u_at[i] + self.slope[i] * (x - (self.lo + i * self.hx))
        return np.broadcast_to(vx[None, None, :], (np.size(z), np.size(y), np.size(x))).copy()


def consistency_data(ncells, lo, hi, k, D, b, c, sigma, seed=0, Dcell=None, field=None, bfield=None):
    """Return (z_star, F) for a seeded random u* in Q_k (all boundary faces Dirichlet).

    Dcell ([ncell, 3, 3], NEXT-1): per-cell tensors for f and the Dirichlet terms of l_h.
    field: any object with eval(x, y, z, d) (default: PolyField of degree k with `seed`).
    bfield: velocity field b(x) (x: (3, npts) -> (3, npts), NEXT-2); default the constant b.
    Quadrature: k+1 Gauss points per direction (exact for polynomial data of the tests)."""
    nc = [int(v) for v in ncells]
    n = k + 1
    D0 = np.asarray(D, float).reshape(3, 3)
    b = np.asarray(b, float)
    h = [(hi[q] - lo[q]) / nc[q] for q in range(3)]
    dT = h[0] * h[1] * h[2]
    xi, w = gauss01(n)
    th, dth = theta(n, xi)          # [point, basis]
    t0, d0 = theta(n, [0.0])
    t1, d1 = theta(n, [1.0])
    u = PolyField(k, lo, hi, seed) if field is None else field
    ncell = nc[0] * nc[1] * nc[2]
    z = np.zeros((ncell, n, n, n))   # [e][jz][jy][jx]
    F = np.zeros((ncell, n, n, n))
    Wv = dT * np.einsum("k,j,i->kji", w, w, w)
    for iz in range(nc[2]):
        for iy in range(nc[1]):
            for ix in range(nc[0]):
                ic = (ix, iy, iz)
                e = ix + nc[0] * (iy + nc[1] * iz)
                D = D0 if Dcell is None else np.asarray(Dcell[e], float).reshape(3, 3)
                X, Y, Zc = _cell_points(lo, h, ic, xi)
                us = u.eval(X, Y, Zc)
                # L2 projection (orthonormal basis, mass = Delta_T I): z_j = (1/Delta_T) int u* phi_j
                z[e] = np.einsum("kji,kc,jb,ia->cba", Wv * us, th, th, th) / dT
                # f = -sum_rs D_rs d_r d_s u* + b . grad u* + c u*
                f = c * us
                bv = _velocity(b, bfield, X, Y, Zc)          # [r][z, y, x]
                for r in range(3):
                    dr = [0, 0, 0]
                    dr[r] += 1
                    f = f + bv[r] * u.eval(X, Y, Zc, tuple(dr))
                    for s in range(3):
                        if D[r, s] != 0.0:
                            drs = [0, 0, 0]
                            drs[r] += 1
                            drs[s] += 1
                            f = f - D[r, s] * u.eval(X, Y, Zc, tuple(drs))
                F[e] += np.einsum("kji,kc,jb,ia->cba", Wv * f, th, th, th)
                # Dirichlet boundary faces
                for q in range(3):
                    for s in (0, 1):
                        if not ((s == 0 and ic[q] == 0) or (s == 1 and ic[q] == nc[q] - 1)):
                            continue
                        nu = np.zeros(3)
                        nu[q] = 1.0 if s == 1 else -1.0
                        gam = (nu @ D @ nu) * sigma
                        pts = [X, Y, Zc]
                        pts[q] = np.array([lo[q] + (ic[q] + s) * h[q]])
                        g = u.eval(*pts)                            # [z,y,x] with size-1 axis q
                        bnu = nu[q] * _velocity(b, bfield, *pts)[q]  # b . nu per face point
                        Wf = dT / h[q] * np.ones_like(g)
                        for r in range(3):
                            if r != q:
                                shape = [1, 1, 1]
                                shape[2 - r] = n
                                Wf = Wf * w.reshape(shape)
                        # per-direction test tables at the face: value and derivative
                        V = [th, th, th]
                        G = [dth, dth, dth]
                        V[q] = t1 if s == 1 else t0
                        G[q] = d1 if s == 1 else d0
                        phi = np.einsum("kc,jb,ia->kjicba", V[2], V[1], V[0])
                        grads = [np.einsum("kc,jb,ia->kjicba", V[2], V[1], G[0]) / h[0],
                                 np.einsum("kc,jb,ia->kjicba", V[2], G[1], V[0]) / h[1],
                                 np.einsum("kc,jb,ia->kjicba", G[2], V[1], V[0]) / h[2]]
                        nDgrad = sum(nu[r2] * D[r2, s2] * grads[s2] for r2 in range(3) for s2 in range(3))
                        phi_in = np.where(bnu >= 0, 0.0, bnu)   # Phi(0, g, b_nu) = b_nu g on inflow
                        integrand = (-phi_in * g + gam * g)[..., None, None, None] * phi \
                            - g[..., None, None, None] * nDgrad
                        F[e] += np.einsum("kji,kjicba->cba", Wf, integrand)
    return z.reshape(-1), F.reshape(-1)


def _velocity(b, bfield, X, Y, Z):
    """b at the tensor grid X (fastest) x Y x Z: array [3][z, y, x]."""
    gz, gy, gx = np.meshgrid(np.atleast_1d(Z), np.atleast_1d(Y), np.atleast_1d(X), indexing="ij")
    if bfield is None:
        return np.stack([np.full(gx.shape, float(b[r])) for r in range(3)])
    pts = np.stack([gx.ravel(), gy.ravel(), gz.ravel()])
    return bfield(pts).reshape((3,) + gx.shape)


def upwind_energy(ncells, lo, hi, k, b, z):
    """1/2 sum_F |b_nu| int_F [[u]]^2 (interior) + 1/2 sum_F |b_nu| int_F u^2 (boundary)."""
    nc = [int(v) for v in ncells]
    n = k + 1
    h = [(hi[q] - lo[q]) / nc[q] for q in range(3)]
    dT = h[0] * h[1] * h[2]
    xi, w = gauss01(n)
    th, _ = theta(n, xi)
    t0, _ = theta(n, [0.0])
    t1, _ = theta(n, [1.0])
    Zc = np.asarray(z, float).reshape(nc[2], nc[1], nc[0], n, n, n)   # [iz][iy][ix][jz][jy][jx]
    E = 0.0
    for q in range(3):
        V1 = [th, th, th]
        V0 = [th, th, th]
        V1[q], V0[q] = t1, t0
        # trace at x_q = 1 and x_q = 0 of every cell at the face Gauss points: [iz,iy,ix, pz,py,px]
        tr1 = np.einsum("ZYXcba,kc,jb,ia->ZYXkji", Zc, V1[2], V1[1], V1[0])
        tr0 = np.einsum("ZYXcba,kc,jb,ia->ZYXkji", Zc, V0[2], V0[1], V0[0])
        wt = np.ones((1, 1, 1))
        for r in range(3):
            shape = [1, 1, 1]
            if r != q:
                shape[2 - r] = n
                wt = wt * w.reshape(shape)
        wt = wt * dT / h[q]
        ax = 2 - q
        lo_sl = [slice(None)] * 3
        hi_sl = [slice(None)] * 3
        lo_sl[ax] = slice(0, -1)
        hi_sl[ax] = slice(1, None)
        jump = tr1[tuple(lo_sl)] - tr0[tuple(hi_sl)]
        E += 0.5 * abs(b[q]) * np.sum(wt * jump ** 2)
        first = [slice(None)] * 3
        last = [slice(None)] * 3
        first[ax] = slice(0, 1)
        last[ax] = slice(-1, None)
        E += 0.5 * abs(b[q]) * np.sum(wt * tr0[tuple(first)] ** 2)
        E += 0.5 * abs(b[q]) * np.sum(wt * tr1[tuple(last)] ** 2)
    return E


def consistency_data_affine(ncells, lo, hi, k, D, b, c, sigma, J, seed=0):
    """(z*, F) on the affinely mapped mesh x = lo + J (xhat - lo) (NEXT-3) for a seeded polynomial u*
    of TOTAL degree min(k, 2) in the physical coordinates (P_k is invariant under affine maps and
    lies in the mapped Q_k, so SIPG reproduces it): u* = a0 + g.x (+ x^T H x for k >= 2).
    Every integral physical: volume |J| dxhat, faces |cof(J) e_q| dShat with nu = cof(J) e_q / |.|,
    l_h of PAPER.md:316-325 on the Dirichlet faces (gamma = nu^T D nu sigma, reading C-6)."""
    nc = [int(v) for v in ncells]
    n = k + 1
    D = np.asarray(D, float).reshape(3, 3)
    b = np.asarray(b, float)
    Jm = np.asarray(J, float).reshape(3, 3)
    detJ = float(np.linalg.det(Jm))
    JinvT = np.linalg.inv(Jm).T
    cof = detJ * JinvT
    lo_v = np.asarray(lo, float)
    rng = np.random.default_rng(seed)
    a0 = rng.uniform(-1, 1)
    g = rng.uniform(-1, 1, 3)
    H = np.zeros((3, 3))
    if k >= 2:
        H = rng.uniform(-1, 1, (3, 3))
        H = 0.5 * (H + H.T)

    def u_star(x):                     # x: (3, npts)
        return a0 + g @ x + np.einsum("ip,ij,jp->p", x, H, x)

    def grad_u(x):
        return g[:, None] + 2.0 * H @ x

    f_const = -2.0 * np.trace(D @ H)   # -div(D grad u*)
    h = [(hi[q] - lo[q]) / nc[q] for q in range(3)]
    dT = h[0] * h[1] * h[2]
    xi, w = gauss01(n)
    th, dth = theta(n, xi)
    t0, d0 = theta(n, [0.0])
    t1, d1 = theta(n, [1.0])
    ncell = nc[0] * nc[1] * nc[2]
    z = np.zeros((ncell, n ** 3))
    F = np.zeros((ncell, n ** 3))

    def phys(ic, pts):                 # tensor points (x fastest) of reference cell ic -> physical (3, npts)
        X = [lo[q] + (ic[q] + np.asarray(pts[q], float)) * h[q] for q in range(3)]
        gz, gy, gx = np.meshgrid(X[2], X[1], X[0], indexing="ij")
        xh = np.stack([gx.ravel(), gy.ravel(), gz.ravel()])
        return lo_v[:, None] + Jm @ (xh - lo_v[:, None])

    def tens(vx, vy, vz):              # [point (z slow, x fast), basis j = jx + n(jy + n jz)]
        return np.einsum("ai,bj,ck->cbakji", vx, vy, vz).reshape(vz.shape[0] * vy.shape[0] * vx.shape[0], -1)

    Wv = dT * np.einsum("k,j,i->kji", w, w, w).reshape(-1)
    phi_v = tens(th, th, th)
    for iz in range(nc[2]):
        for iy in range(nc[1]):
            for ix in range(nc[0]):
                ic = (ix, iy, iz)
                e = ix + nc[0] * (iy + nc[1] * iz)
                x = phys(ic, [xi, xi, xi])
                us = u_star(x)
                z[e] = (Wv * us) @ phi_v / dT                    # (1/(|J| dT)) int u* phi |J| dxhat
                fv = f_const + b @ grad_u(x) + c * us
                F[e] += detJ * (Wv * fv) @ phi_v
                for q in range(3):
                    for s in (0, 1):
                        if not ((s == 0 and ic[q] == 0) or (s == 1 and ic[q] == nc[q] - 1)):
                            continue
                        eq = np.zeros(3)
                        eq[q] = 1.0
                        area = float(np.linalg.norm(cof @ eq))
                        nu = (cof @ eq) / area * (1.0 if s == 1 else -1.0)      # outward physical normal
                        pts = [xi, xi, xi]
                        pts[q] = np.array([float(s)])
                        xf = phys(ic, pts)
                        gval = u_star(xf)
                        V = [th, th, th]
                        G = [dth, dth, dth]
                        V[q] = t1 if s == 1 else t0
                        G[q] = d1 if s == 1 else d0
                        phi = tens(V[0], V[1], V[2])
                        grads = np.stack([tens(G[0], V[1], V[2]) / h[0], tens(V[0], G[1], V[2]) / h[1],
                                          tens(V[0], V[1], G[2]) / h[2]])   # reference-mesh gradients
                        pg = np.einsum("rs,spj->rpj", JinvT, grads)         # physical gradients
                        nDg = np.einsum("r,rs,spj->pj", nu, D, pg)
                        Wf = area * dT / h[q] * np.einsum("a,b->ba", w, w).reshape(-1)
                        bnu = b @ nu
                        gam = (nu @ D @ nu) * sigma
                        phi_in = 0.0 if bnu >= 0 else bnu                  # Phi(0, g, b_nu)
                        F[e] += ((-phi_in + gam) * Wf * gval) @ phi - (Wf * gval) @ nDg
    return z.reshape(-1), F.reshape(-1)
