"""O-2: the system matrix A_ij = a_h(phi_j, phi_i) assembled entry by entry from
the weak form (numpy, dense, tiny meshes). TEST INFRASTRUCTURE ONLY.

Definitions followed:
  (A_h)_ij = a_h(phi_j, phi_i)
  a_h(u,v) = sum_T [(D grad u - b u, grad v)_T + (c u, v)_T]
           + sum_{F interior} (Phi(u-,u+,nu.b), [[v]])_F
           + sum_{F boundary, Dirichlet/outflow} (Phi(u,0,nu.b), v)_F
           - sum_{F in iD} (nu.{D grad u}_w, [[v]])_F
           - sum_{F in iD} (nu.{D grad v}_w, [[u]])_F
           + sum_{F in iD} gamma_F ([[u]], [[v]])_F                 eq:blf
  [[v]] = v- - v+, {v}_w = w- v- + w+ v+ (reading C-1 of PAPER.md:271),
  on the boundary [[v]] = {v}_w = v-                              PAPER.md:282-286
  w- = d+/(d- + d+), w+ = d-/(d- + d+), d = nu^T D nu
  gamma_F = <d-, d+> * sigma (reading C-4), boundary d * sigma (C-6)
  Phi(u-,u+,b_nu) = b_nu u- if b_nu >= 0 else b_nu u+             PAPER.md:334-341

Every face integral is written as a bilinear form over the COMBINED trial and
test spaces of the two adjacent cells, evaluated at the tensor Gauss points of
the face, and scattered into the global matrix. No sum factorization, no
splitting into the per-cell formulas used by O-1.

NEXT-1 (the paper's Problem A): `periodic[q]` glues the two box
sides normal to q (the wrap face is an interior face, T- = the last cell, nu = +e_q);
`Dcell[e]` gives cell e its own tensor, so D-, D+, the weights w+- and the harmonic
penalty <d-, d+> differ per face.

NEXT-2/3 (the Taylor-Green run): `m` Gauss points per direction
(over-integration, q = 2p+4 -> m = k+3) and a velocity field `bfield(x) -> b` evaluated at
every quadrature point of volumes and faces.

NEXT-3 affine geometry (Problem B's "affine geometries"): `J` maps the
axis-aligned reference mesh on [lo, hi] to the physical mesh x = lo + J (xhat - lo). Every
integral is evaluated in PHYSICAL terms: gradients J^-T grad_hat, volume element |J| dxhat,
face normals nu = cof(J) e_q / |cof(J) e_q| and surface element |cof(J) e_q| dShat (cof(J) =
|J| J^-T), delta = nu^T D nu and b.nu with the physical normal, the penalty sigma as given.
"""
import numpy as np

from .tables import gauss01, theta

VOLUME, INTERIOR, BOUNDARY, ALL = 1, 2, 4, 7


def _cell_index(ix, iy, iz, nc):
    return ix + nc[0] * (iy + nc[1] * iz)


def _tensor(vals):
    """phi_j(p) for j = jx + n(jy + n jz), p = px + m(py + m pz), from per-direction tables vals[q][p_q, j_q]."""
    vx, vy, vz = vals
    # out[pz,py,px,jz,jy,jx]
    out = np.einsum("ai,bj,ck->cbakji", vx, vy, vz)
    mz, my, mx = vz.shape[0], vy.shape[0], vx.shape[0]
    n3 = vx.shape[1] * vy.shape[1] * vz.shape[1]
    return out.reshape(mz * my * mx, n3)


def _basis_on(n, pts_per_dir, h):
    """Values [p, j] and physical gradients [r, p, j] of all cell basis functions
    at the tensor point set pts_per_dir[q] (reference coordinates)."""
    tabs = [theta(n, pts_per_dir[q]) for q in range(3)]
    V = [t[0] for t in tabs]
    G = [t[1] for t in tabs]
    phi = _tensor(V)
    grad = np.stack([
        _tensor([G[0], V[1], V[2]]) / h[0],
        _tensor([V[0], G[1], V[2]]) / h[1],
        _tensor([V[0], V[1], G[2]]) / h[2],
    ])
    return phi, grad


def taylor_green(x):
    """eq:2: x of shape (3, npts) -> b of shape (3, npts)."""
    return np.stack([np.cos(x[0]) * np.sin(-x[1]) * np.sin(-x[2]),
                     0.5 * np.sin(x[0]) * np.cos(-x[1]) * np.sin(-x[2]),
                     0.5 * np.sin(x[0]) * np.sin(-x[1]) * np.cos(-x[2])])


def linear_field(x):
    """The linear divergence-free test field b = (x2, x3, x1)."""
    return np.stack([x[1], x[2], x[0]])


def assemble(ncells, lo, hi, k, D, b, c, sigma, mask=ALL, avg_sign=1.0, periodic=(0, 0, 0), Dcell=None, m=0,
             bfield=None, J=None):
    """Dense A (N x N), N = prod(ncells) * (k+1)^3, cell-major global order (C-3).

    avg_sign = -1 selects the weighted average exactly as PAPER.md:271 prints it
    ({v}_w = w- v- - w+ v+); used only by the test that shows this reading is
    inconsistent (reading C-1). The oracle's operator is avg_sign = +1.
    periodic / Dcell ([ncell, 3, 3]): NEXT-1, see the module docstring."""
    nc = [int(v) for v in ncells]
    n = k + 1
    n3 = n ** 3
    b = np.asarray(b, dtype=np.float64)
    ncell0 = nc[0] * nc[1] * nc[2]
    if Dcell is None:
        Dcell = np.tile(np.asarray(D, dtype=np.float64).reshape(1, 3, 3), (ncell0, 1, 1))
    Dcell = np.asarray(Dcell, dtype=np.float64).reshape(ncell0, 3, 3)
    h = [(hi[q] - lo[q]) / nc[q] for q in range(3)]
    dT = h[0] * h[1] * h[2]
    ncell = nc[0] * nc[1] * nc[2]
    A = np.zeros((ncell * n3, ncell * n3))
    m = m if m else n
    xi, w = gauss01(m)
    Jm = np.eye(3) if J is None else np.asarray(J, dtype=np.float64).reshape(3, 3)
    detJ = float(np.linalg.det(Jm))
    if detJ <= 0:
        raise ValueError("the affine map must preserve orientation")
    JinvT = np.linalg.inv(Jm).T
    cof = detJ * JinvT
    lo_v = np.asarray(lo, dtype=np.float64)

    def phys_grad(grad):
        """reference-mesh gradients (3, p, j) -> physical gradients J^-T grad_hat."""
        return np.einsum("rs,spj->rpj", JinvT, grad)

    def points(ic, pts_per_dir):
        """physical coordinates (3, npts) of the tensor point set, x fastest (as _tensor orders it)."""
        X = [lo[q] + (ic[q] + np.asarray(pts_per_dir[q], float)) * h[q] for q in range(3)]
        gz, gy, gx = np.meshgrid(X[2], X[1], X[0], indexing="ij")
        xhat = np.stack([gx.ravel(), gy.ravel(), gz.ravel()])
        return lo_v[:, None] + Jm @ (xhat - lo_v[:, None])     # physical points

    def velocity(ic, pts_per_dir):
        npts = np.prod([np.size(v) for v in pts_per_dir])
        if bfield is None:
            return np.tile(b[:, None], (1, npts))
        return bfield(points(ic, pts_per_dir))

    # ---- volume blocks (coefficients constant per cell, uniform cells)
    if mask & VOLUME:
        phi, grad = _basis_on(n, [xi, xi, xi], h)
        grad = phys_grad(grad)
        W = detJ * dT * np.einsum("a,b,c->cba", w, w, w).reshape(-1)
        for e in range(ncell):
            ic = (e % nc[0], (e // nc[0]) % nc[1], e // (nc[0] * nc[1]))
            bp = velocity(ic, [xi, xi, xi])                       # (3, npts)
            # integrand (D grad u - b u) . grad v + c u v, u = phi_j (columns), v = phi_i (rows)
            flux = np.einsum("rs,spj->rpj", Dcell[e], grad) - bp[:, :, None] * phi[None, :, :]
            Avol = np.einsum("p,rpi,rpj->ij", W, grad, flux) + c * np.einsum("p,pi,pj->ij", W, phi, phi)
            A[e * n3:(e + 1) * n3, e * n3:(e + 1) * n3] += Avol

    # ---- faces
    for q in range(3):
        t = [r for r in range(3) if r != q]
        dF = dT / h[q]
        eq = np.zeros(3)
        eq[q] = 1.0
        area = float(np.linalg.norm(cof @ eq))              # |cof(J) e_q|: physical / reference face measure
        Wf = area * dF * np.einsum("a,b->ba", w, w).reshape(-1)   # tangential point p = pt1 + m*pt2
        nu = (cof @ eq) / area                              # physical unit normal of a reference q-face

        def face_basis(s):
            pts = [None, None, None]
            pts[q] = np.array([float(s)])
            pts[t[0]] = xi
            pts[t[1]] = xi
            phi, grad = _basis_on(n, pts, h)
            return phi, phys_grad(grad)   # point ordering x-fastest over the three dirs = t1-fastest over the face

        phi1, grad1 = face_basis(1)   # face x_q = 1 of a cell
        phi0, grad0 = face_basis(0)   # face x_q = 0 of a cell

        for iz in range(nc[2]):
            for iy in range(nc[1]):
                for ix in range(nc[0]):
                    ic = [ix, iy, iz]
                    e = _cell_index(ix, iy, iz, nc)
                    # interior face with this cell as T- (low side) and its +q neighbour as T+
                    if (ic[q] + 1 < nc[q] or periodic[q]) and (mask & INTERIOR):
                        jc = list(ic)
                        jc[q] = (jc[q] + 1) % nc[q]
                        f = _cell_index(jc[0], jc[1], jc[2], nc)
                        Dm, Dp = Dcell[e], Dcell[f]
                        npts = phi1.shape[0]
                        Z = np.zeros((npts, n3))
                        um = np.hstack([phi1, Z])              # u- of combined trial [T- dofs, T+ dofs]
                        up = np.hstack([Z, phi0])              # u+
                        gm = np.concatenate([grad1, np.zeros_like(grad1)], axis=2)
                        gp = np.concatenate([np.zeros_like(grad0), grad0], axis=2)
                        dm, dp = nu @ Dm @ nu, nu @ Dp @ nu
                        if dm + dp == 0.0:
                            wm = wp = 0.5
                        else:
                            wm, wp = dp / (dm + dp), dm / (dm + dp)
                        gam = (0.0 if dm + dp == 0.0 else 2 * dm * dp / (dm + dp)) * sigma
                        fpts = [None, None, None]
                        fpts[q], fpts[t[0]], fpts[t[1]] = np.array([1.0]), xi, xi
                        bnu = (velocity(ic, fpts).T @ nu)[:, None]        # b . nu per face point
                        Phi = np.where(bnu >= 0, bnu * um, bnu * up)      # linear in the trial function
                        nDg = (wm * np.einsum("r,rs,spj->pj", nu, Dm, gm)
                               + avg_sign * wp * np.einsum("r,rs,spj->pj", nu, Dp, gp))   # nu.{D grad .}_w
                        jump = um - up
                        # rows: test functions (same combined space), columns: trial functions
                        B = (np.einsum("p,pi,pj->ij", Wf, jump, Phi)
                             - np.einsum("p,pi,pj->ij", Wf, jump, nDg)
                             - np.einsum("p,pi,pj->ij", Wf, nDg, jump)
                             + gam * np.einsum("p,pi,pj->ij", Wf, jump, jump))
                        # scatter the 2x2 blocks (e == f when a periodic direction has one cell)
                        for bi, ci in ((0, e), (1, f)):
                            for bj, cj in ((0, e), (1, f)):
                                A[ci * n3:(ci + 1) * n3, cj * n3:(cj + 1) * n3] += \
                                    B[bi * n3:(bi + 1) * n3, bj * n3:(bj + 1) * n3]
                    # boundary faces of this cell in direction q
                    if mask & BOUNDARY:
                        for s in (0, 1):
                            if not periodic[q] and ((s == 0 and ic[q] == 0) or (s == 1 and ic[q] == nc[q] - 1)):
                                D = Dcell[e]
                                phs, grs = (phi1, grad1) if s == 1 else (phi0, grad0)
                                nuo = nu * (1.0 if s == 1 else -1.0)
                                fpts = [None, None, None]
                                fpts[q], fpts[t[0]], fpts[t[1]] = np.array([float(s)]), xi, xi
                                bnu = (velocity(ic, fpts).T @ nuo)[:, None]
                                Phi = np.where(bnu >= 0, bnu * phs, 0.0)         # Phi(u, 0, b_nu)
                                sn = np.einsum("r,rs,spj->pj", nuo, D, grs)     # nu.D grad
                                gam = (nuo @ D @ nuo) * sigma
                                B = (np.einsum("p,pi,pj->ij", Wf, phs, Phi)
                                     - np.einsum("p,pi,pj->ij", Wf, phs, sn)
                                     - np.einsum("p,pi,pj->ij", Wf, sn, phs)
                                     + gam * np.einsum("p,pi,pj->ij", Wf, phs, phs))
                                sl = slice(e * n3, (e + 1) * n3)
                                A[sl, sl] += B
    return A
