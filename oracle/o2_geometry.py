"""O-2 on multilinear (Q1) meshes: A_ij = a_h(phi_j, phi_i) assembled entry by entry from the
weak form with the geometry evaluated at every quadrature point (numpy, dense, tiny meshes).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's Problem C has "multilinear geometries": "the transformation
x = mu_T(xhat) from the reference element That to the real element T is a d-valued Q_1 finite
element function". Here:

  mu_T(xi) = sum_{c in {0,1}^3} X_c prod_q B_{c_q}(xi_q),  B_0(t) = 1 - t, B_1(t) = t,
  xi in [0,1]^3 the cell's reference coordinates, X_c the 8 vertices of the cell in a structured
  vertex grid X[iz][iy][ix] (cell (ix, iy, iz) has the corners X[iz+c2][iy+c1][ix+c0]);
  J(xi) = d mu / d xi (J_rs = dx_r / dxi_s), basis phi_j(x) = theta_j(mu^-1(x)) (reading C-2),
  grad phi = J^-T gradhat phi, dx = det J dxi;
  on the face xi_q = s: the tangent vectors t_a = d mu / d xi_a, the surface normal
  N = t_{q+1} x t_{q+2} (indices cyclic; the cofactor column cof(J) e_q, pointing to +xi_q),
  dS = |N| dxi_t1 dxi_t2, the unit normal nu = N / |N|.

Every term of eq:blf as in o2_assembled.py: the face integral is a bilinear
form over the COMBINED trial and test spaces of the two cells, each side's gradients with ITS
OWN Jacobian at the common face points (a conforming structured mesh: both cells parametrise the
shared face by the same (xi_t1, xi_t2)); delta = nu^T D nu, w+- = d-+/(d- + d+) (= 1/2 for a
constant D), gamma = <d-, d+> sigma (reading C-4 / N-7: sigma is the one input number),
Phi = upwind b.nu. Periodic directions: the wrap neighbour is the cell at the
other end (its vertices; the Jacobian does not see the period's translation). Quadrature: m
Gauss points per direction (m = k+1: q = 2p; Problem C's q = 3p+4: m = ceil((3k+5)/2)), the same
rule on volumes and faces; the integrands are rational in xi (1 / det J), so the operator is
that of this rule, exactly what the kernel evaluates.
"""
import numpy as np

from .tables import gauss01, theta

VOLUME, INTERIOR, BOUNDARY, ALL = 1, 2, 4, 7


def corners(X, ic):
    """The 8 vertices [c2][c1][c0][3] of cell ic = (ix, iy, iz) of the vertex grid X[iz][iy][ix][3]."""
    ix, iy, iz = ic
    return X[iz:iz + 2, iy:iy + 2, ix:ix + 2]


def q1_map(C, pts):
    """x = mu(xi) and J = d mu / d xi at reference points pts (npts, 3) for corners C [c2][c1][c0][3]."""
    pts = np.asarray(pts, float)
    B = [np.stack([1.0 - pts[:, q], pts[:, q]]) for q in range(3)]     # [c_q][p]
    dB = [np.stack([-np.ones(len(pts)), np.ones(len(pts))]) for q in range(3)]
    x = np.einsum("zyxr,zp,yp,xp->pr", C, B[2], B[1], B[0])
    J = np.stack([np.einsum("zyxr,zp,yp,xp->pr", C, B[2], B[1], dB[0]),
                  np.einsum("zyxr,zp,yp,xp->pr", C, B[2], dB[1], B[0]),
                  np.einsum("zyxr,zp,yp,xp->pr", C, dB[2], B[1], B[0])], axis=2)   # J[p][r][s] = dx_r/dxi_s
    return x, J


def _tensor_pts(pts_per_dir):
    """Reference points (npts, 3), x fastest, of the tensor set pts_per_dir[q]."""
    gz, gy, gx = np.meshgrid(pts_per_dir[2], pts_per_dir[1], pts_per_dir[0], indexing="ij")
    return np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)


def _basis(n, pts_per_dir):
    """phi [p, j] and reference gradients [s, p, j] (j = jx + n(jy + n jz)) on the tensor set."""
    tabs = [theta(n, pts_per_dir[q]) for q in range(3)]
    V = [t[0] for t in tabs]
    G = [t[1] for t in tabs]

    def tens(vx, vy, vz):
        out = np.einsum("ai,bj,ck->cbakji", vx, vy, vz)
        return out.reshape(vz.shape[0] * vy.shape[0] * vx.shape[0], -1)
    return tens(V[0], V[1], V[2]), np.stack([tens(G[0], V[1], V[2]), tens(V[0], G[1], V[2]),
                                             tens(V[0], V[1], G[2])])


def _phys_grad(J, gref):
    """grad phi = J^-T gradhat phi at every point: gref [s, p, j] -> [r, p, j]."""
    JinvT = np.linalg.inv(J).transpose(0, 2, 1)                      # [p][r][s]
    return np.einsum("prs,spj->rpj", JinvT, gref)


def _bil(W, a, b):
    """sum_p W_p a_pi b_pj (a quadrature-weighted bilinear form; numpy matmul)."""
    return (a * W[:, None]).T @ b


def face_normal(J, q):
    """N = t_{q+1} x t_{q+2} (cyclic) at each point: the area-weighted normal towards +xi_q."""
    a, b = (q + 1) % 3, (q + 2) % 3
    return np.cross(J[:, :, a], J[:, :, b])


def assemble(ncells, X, k, D, b, c, sigma, m=0, periodic=(0, 0, 0), mask=ALL):
    """Dense A (cell-major order, C-3) on the multilinear mesh with vertex grid X[iz][iy][ix][3]
    ((N2+1) x (N1+1) x (N0+1) vertices)."""
    nc = [int(v) for v in ncells]
    n = k + 1
    n3 = n ** 3
    m = m if m else n
    D = np.asarray(D, float).reshape(3, 3)
    b = np.asarray(b, float)
    X = np.asarray(X, float)
    assert X.shape == (nc[2] + 1, nc[1] + 1, nc[0] + 1, 3)
    ncell = nc[0] * nc[1] * nc[2]
    A = np.zeros((ncell * n3, ncell * n3))
    xi, w = gauss01(m)

    def cid(ic):
        return ic[0] + nc[0] * (ic[1] + nc[1] * ic[2])

    # ---- volume: (D grad u - b u, grad v)_T + (c u, v)_T
    if mask & VOLUME:
        pts = _tensor_pts([xi, xi, xi])
        phi, gref = _basis(n, [xi, xi, xi])
        wv = np.einsum("c,b,a->cba", w, w, w).reshape(-1)
        for iz in range(nc[2]):
            for iy in range(nc[1]):
                for ix in range(nc[0]):
                    ic = (ix, iy, iz)
                    _, J = q1_map(corners(X, ic), pts)
                    det = np.linalg.det(J)
                    assert np.all(det > 0), "inverted cell"
                    grad = _phys_grad(J, gref)
                    W = wv * det
                    flux = np.einsum("rs,spj->rpj", D, grad) - b[:, None, None] * phi[None]
                    e = cid(ic)
                    A[e * n3:(e + 1) * n3, e * n3:(e + 1) * n3] += (
                        sum(_bil(W, grad[r], flux[r]) for r in range(3)) + c * _bil(W, phi, phi))

    # ---- faces
    for q in range(3):
        t = [r for r in range(3) if r != q]
        wf = np.einsum("b,a->ba", w, w).reshape(-1)          # point pt1 + m pt2 (t1 fastest)

        def side(s):
            pp = [None, None, None]
            pp[q] = np.array([float(s)])
            pp[t[0]], pp[t[1]] = xi, xi
            phi, gref = _basis(n, pp)
            return _tensor_pts(pp), phi, gref

        pts1, phi1, gref1 = side(1)          # face xi_q = 1 of a cell (it is T-)
        pts0, phi0, gref0 = side(0)          # face xi_q = 0 (T+)
        for iz in range(nc[2]):
            for iy in range(nc[1]):
                for ix in range(nc[0]):
                    ic = [ix, iy, iz]
                    e = cid(ic)
                    _, Jm1 = q1_map(corners(X, ic), pts1)
                    N1 = face_normal(Jm1, q)
                    if (ic[q] + 1 < nc[q] or periodic[q]) and (mask & INTERIOR):
                        jc = list(ic)
                        jc[q] = (jc[q] + 1) % nc[q]
                        f = cid(jc)
                        _, Jp0 = q1_map(corners(X, jc), pts0)
                        area = np.linalg.norm(N1, axis=1)
                        nu = N1 / area[:, None]
                        Wf = wf * area
                        npts = phi1.shape[0]
                        Z = np.zeros((npts, n3))
                        um, up = np.hstack([phi1, Z]), np.hstack([Z, phi0])
                        gm = _phys_grad(Jm1, gref1)
                        gp = _phys_grad(Jp0, gref0)
                        gm = np.concatenate([gm, np.zeros_like(gm)], axis=2)
                        gp = np.concatenate([np.zeros_like(gp), gp], axis=2)
                        d = np.einsum("pr,rs,ps->p", nu, D, nu)           # d- = d+ (one tensor)
                        wm = wp = 0.5
                        gam = d * sigma                                    # <d, d> = d
                        bnu = (nu @ b)[:, None]
                        Phi = np.where(bnu >= 0, bnu * um, bnu * up)
                        nDg = wm * np.einsum("pr,rs,spj->pj", nu, D, gm) + wp * np.einsum("pr,rs,spj->pj", nu, D, gp)
                        jump = um - up
                        B = (_bil(Wf, jump, Phi) - _bil(Wf, jump, nDg) - _bil(Wf, nDg, jump)
                             + _bil(Wf * gam, jump, jump))
                        for bi, ci in ((0, e), (1, f)):
                            for bj, cj in ((0, e), (1, f)):
                                A[ci * n3:(ci + 1) * n3, cj * n3:(cj + 1) * n3] += \
                                    B[bi * n3:(bi + 1) * n3, bj * n3:(bj + 1) * n3]
                    if mask & BOUNDARY and not periodic[q]:
                        for s in (0, 1):
                            if not ((s == 0 and ic[q] == 0) or (s == 1 and ic[q] == nc[q] - 1)):
                                continue
                            if s == 1:
                                Jb, phs, grf, N = Jm1, phi1, gref1, N1
                            else:
                                _, Jb = q1_map(corners(X, ic), pts0)
                                phs, grf, N = phi0, gref0, -face_normal(Jb, q)   # outward: towards -xi_q
                            area = np.linalg.norm(N, axis=1)
                            nuo = N / area[:, None]
                            Wf = wf * area
                            grs = _phys_grad(Jb, grf)
                            bnu = (nuo @ b)[:, None]
                            Phi = np.where(bnu >= 0, bnu * phs, 0.0)
                            sn = np.einsum("pr,rs,spj->pj", nuo, D, grs)
                            gam = np.einsum("pr,rs,ps->p", nuo, D, nuo) * sigma
                            B = (_bil(Wf, phs, Phi) - _bil(Wf, phs, sn) - _bil(Wf, sn, phs)
                                 + _bil(Wf * gam, phs, phs))
                            A[e * n3:(e + 1) * n3, e * n3:(e + 1) * n3] += B
    return A


def consistency_data(ncells, X, k, D, b, c, sigma, m=0, seed=0):
    """(z*, F) for the physical linear field u*(x) = a0 + g.x on the multilinear mesh (all faces
    Dirichlet, g_D = u*): u* o mu_T is Q_1 in xi, so z*_j = int_[0,1]^3 (u* o mu) theta_j dxi is its
    exact representation; f = -div(D grad u*) + b.grad u* + c u* = b.g + c u*; F = l_h(phi_i)
     on the physical mesh with this rule. A z* = F holds to rounding once the
    rule integrates the (then polynomial) integrands exactly: 2m - 1 >= k + 3."""
    nc = [int(v) for v in ncells]
    n = k + 1
    m = m if m else n
    D = np.asarray(D, float).reshape(3, 3)
    b = np.asarray(b, float)
    rng = np.random.default_rng(seed)
    a0, g = rng.uniform(-1, 1), rng.uniform(-1, 1, 3)
    xi, w = gauss01(m)
    pts = _tensor_pts([xi, xi, xi])
    phi, _ = _basis(n, [xi, xi, xi])
    wv = np.einsum("c,b,a->cba", w, w, w).reshape(-1)
    ncell = nc[0] * nc[1] * nc[2]
    z = np.zeros((ncell, n ** 3))
    F = np.zeros((ncell, n ** 3))
    wf = np.einsum("b,a->ba", w, w).reshape(-1)
    for iz in range(nc[2]):
        for iy in range(nc[1]):
            for ix in range(nc[0]):
                ic = (ix, iy, iz)
                e = ix + nc[0] * (iy + nc[1] * iz)
                C = corners(X, ic)
                x, J = q1_map(C, pts)
                us = a0 + x @ g
                z[e] = (wv * us) @ phi
                F[e] += (wv * np.linalg.det(J) * (b @ g + c * us)) @ phi
                for q in range(3):
                    t = [r for r in range(3) if r != q]
                    for s in (0, 1):
                        if not ((s == 0 and ic[q] == 0) or (s == 1 and ic[q] == nc[q] - 1)):
                            continue
                        pp = [None, None, None]
                        pp[q] = np.array([float(s)])
                        pp[t[0]], pp[t[1]] = xi, xi
                        fp = _tensor_pts(pp)
                        phs, grf = _basis(n, pp)
                        xf, Jf = q1_map(C, fp)
                        N = face_normal(Jf, q) * (1.0 if s == 1 else -1.0)
                        area = np.linalg.norm(N, axis=1)
                        nuo = N / area[:, None]
                        Wf = wf * area
                        gval = a0 + xf @ g
                        nDg = np.einsum("pr,rs,spj->pj", nuo, D, _phys_grad(Jf, grf))
                        bnu = nuo @ b
                        gam = np.einsum("pr,rs,ps->p", nuo, D, nuo) * sigma
                        phi_in = np.where(bnu >= 0, 0.0, bnu)                    # Phi(0, g, b_nu)
                        F[e] += ((-phi_in + gam) * Wf * gval) @ phs - (Wf * gval) @ nDg
    return z.reshape(-1), F.reshape(-1)
