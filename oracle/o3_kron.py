"""O-3: Kronecker closed form of the operator for DIAGONAL constant D, constant b, c
on a structured box of uniform cuboid cells. TEST INFRASTRUCTURE ONLY.

Why it holds: with constant diagonal D, b, c every term of a_h (eq:blf,
PAPER.md:301-315) factorizes across directions, and the orthonormal 1D
mass matrix on a cell of size h is h*I, so

    A = sum_q (prod_{r != q} h_r) * (I x .. x L_q x .. x I) + c * Delta_T * I,

where L_q is the block-tridiagonal 1D operator along direction q acting on
the line index X = e*n + j (cell e along q, local 1D index j).

1D reference integrals on [0,1] for theta_j = sqrt(2j+1) P_j(2x-1), derived in
closed form (test index i = row, trial index j = column):
  K_ij = int theta'_i theta'_j = 2 sqrt((2i+1)(2j+1)) min(i,j)(min(i,j)+1)  if i+j even, else 0
  C_ij = int theta'_i theta_j  = 2 sqrt((2i+1)(2j+1))                      if i>j and i+j odd, else 0
  theta_j(1) = sqrt(2j+1), theta_j(0) = (-1)^j sqrt(2j+1)
  theta'_j(1) = sqrt(2j+1) j(j+1), theta'_j(0) = (-1)^(j+1) sqrt(2j+1) j(j+1)
1D blocks of L_q (f1 = D_qq theta'(1)/h_q, f0 = D_qq theta'(0)/h_q, gamma = D_qq sigma,
w = 1/2 for constant D, Phi upwind by sign of b_q; outer products row (test) x col (trial)):
  cell e:              (D_qq/h_q) K - b_q C                            volume term
  interior e|e+1, T- = e, nu = +e_q:
    [e,e]     += [b>=0] b t1t1 - 1/2 t1 f1 - 1/2 f1 t1 + gamma t1 t1
    [e,e+1]   += [b<0]  b t1t0 - 1/2 t1 f0 + 1/2 f1 t0 - gamma t1 t0
    [e+1,e]   += -[b>=0] b t0t1 + 1/2 t0 f1 - 1/2 f0 t1 - gamma t0 t1
    [e+1,e+1] += -[b<0]  b t0t0 + 1/2 t0 f0 + 1/2 f0 t0 + gamma t0 t0
  boundary x=0 of cell 0 (nu = -1, fn = -f0): [0,0] += [-b>=0](-b) t0t0 - t0 fn - fn t0 + gamma t0t0
  boundary x=1 of cell N-1 (nu = +1):         [N-1,N-1] += [b>=0] b t1t1 - t1 f1 - f1 t1 + gamma t1t1
(These are the 1D restrictions of the volume, upwind, consistency, symmetry and
penalty terms of eq:blf; the derivation is written out in DESIGN.md.)
"""
import numpy as np
import scipy.sparse as sp

VOLUME, INTERIOR, BOUNDARY, ALL = 1, 2, 4, 7


def ref_1d(n):
    j = np.arange(n)
    s = np.sqrt(2.0 * j + 1.0)
    I, J = np.meshgrid(j, j, indexing="ij")
    mn = np.minimum(I, J)
    K = np.where((I + J) % 2 == 0, 2.0 * np.outer(s, s) * mn * (mn + 1), 0.0)
    C = np.where((I > J) & ((I + J) % 2 == 1), 2.0 * np.outer(s, s), 0.0)
    t1 = s.copy()
    t0 = ((-1.0) ** j) * s
    d1 = s * j * (j + 1)
    d0 = ((-1.0) ** (j + 1)) * s * j * (j + 1)
    return K, C, t0, t1, d0, d1


def line_operator(N, n, h, Dqq, bq, sigma, mask=ALL, periodic=False):
    """Sparse (N n) x (N n) 1D operator L_q. periodic: the face between cell N-1 (T-) and
    cell 0 (T+) is an interior face with the same blocks (NEXT-1)."""
    K, C, t0, t1, d0, d1 = ref_1d(n)
    f1, f0 = Dqq * d1 / h, Dqq * d0 / h
    gam = Dqq * sigma
    o = np.outer
    blocks = {}

    def add(a, c, B):
        blocks[(a, c)] = blocks.get((a, c), 0.0) + B

    for e in range(N):
        if mask & VOLUME:
            add(e, e, (Dqq / h) * K - bq * C)
        if (mask & INTERIOR) and (e + 1 < N or periodic):
            up = 1.0 if bq >= 0 else 0.0
            dn = 1.0 - up
            e1 = (e + 1) % N
            add(e, e, up * bq * o(t1, t1) - 0.5 * o(t1, f1) - 0.5 * o(f1, t1) + gam * o(t1, t1))
            add(e, e1, dn * bq * o(t1, t0) - 0.5 * o(t1, f0) + 0.5 * o(f1, t0) - gam * o(t1, t0))
            add(e1, e, -up * bq * o(t0, t1) + 0.5 * o(t0, f1) - 0.5 * o(f0, t1) - gam * o(t0, t1))
            add(e1, e1, -dn * bq * o(t0, t0) + 0.5 * o(t0, f0) + 0.5 * o(f0, t0) + gam * o(t0, t0))
    if (mask & BOUNDARY) and not periodic:
        fn = -f0
        bl = -bq
        add(0, 0, (bl if bl >= 0 else 0.0) * o(t0, t0) - o(t0, fn) - o(fn, t0) + gam * o(t0, t0))
        add(N - 1, N - 1, (bq if bq >= 0 else 0.0) * o(t1, t1) - o(t1, f1) - o(f1, t1) + gam * o(t1, t1))
    rows, cols, vals = [], [], []
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    for (a, c), B in blocks.items():
        B = np.broadcast_to(B, (n, n))
        rows.append((a * n + ii).ravel())
        cols.append((c * n + jj).ravel())
        vals.append(np.asarray(B).ravel())
    if not rows:
        return sp.csr_matrix((N * n, N * n))
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(N * n, N * n))


def apply(ncells, lo, hi, k, D, b, c, sigma, z, mask=ALL, periodic=(0, 0, 0)):
    """y = A z for diagonal D (raises for off-diagonal D). z, y cell-major (C-3).
    periodic[q]: glue the sides normal to q (NEXT-1)."""
    D = np.asarray(D, dtype=np.float64).reshape(3, 3)
    if np.any(D - np.diag(np.diag(D))):
        raise ValueError("O-3 covers diagonal D only")
    nx, ny, nz = (int(v) for v in ncells)
    n = k + 1
    h = [(hi[q] - lo[q]) / ncells[q] for q in range(3)]
    dT = h[0] * h[1] * h[2]
    # cell-major [iz][iy][ix][jz][jy][jx] -> global lines [iz jz][iy jy][ix jx]
    Z = np.asarray(z, dtype=np.float64).reshape(nz, ny, nx, n, n, n).transpose(0, 3, 1, 4, 2, 5)
    Z = np.ascontiguousarray(Z).reshape(nz * n, ny * n, nx * n)
    Y = np.zeros_like(Z)
    # the 1D volume, upwind and penalty terms are all in L_q; the mass terms of
    # the other directions give the factor dT / h_q
    lmask = mask & (INTERIOR | BOUNDARY | VOLUME)
    for q, (N, axis) in enumerate(((nx, 2), (ny, 1), (nz, 0))):
        L = line_operator(N, n, h[q], D[q, q], b[q], sigma, lmask, bool(periodic[q]))
        fac = dT / h[q]
        Zm = np.moveaxis(Z, axis, -1)
        shp = Zm.shape
        R = (L @ Zm.reshape(-1, shp[-1]).T).T.reshape(shp)
        Y += fac * np.moveaxis(R, -1, axis)
    if mask & VOLUME:
        Y += c * dT * Z
    Y = Y.reshape(nz, n, ny, n, nx, n).transpose(0, 2, 4, 1, 3, 5)
    return np.ascontiguousarray(Y).reshape(-1)
