"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle
tests. Holds none of the method's arithmetic (no basis, quadrature or flux).

z is i.i.d. uniform[-1,1] FP64 drawn by a counter-based splitmix64 over the
GLOBAL cell-major DOF index g (reading C-13), all arithmetic mod 2^64:

    x = (seed << 40) + g + 0x9E3779B97F4A7C15
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9
    x = (x ^ (x >> 27)) * 0x94D049BB133111EB
    x ^= x >> 31
    z = (x >> 11) * 2^-53 * 2 - 1

The same generator exists as a CUDA kernel in the library (dg_fill_uniform,
paper_1711_10885_b200/csrc/dg_aux.cu) so multi-GB inputs can be produced in
HBM; tests check the two bit for bit. It is exact in FP64 and independent of
the partition, so a rank can generate its own block from global indices.
"""
import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def uniform_from_index(g, seed):
    """Values for an array of global indices g (uint64-convertible)."""
    with np.errstate(over="ignore"):
        x = np.asarray(g, dtype=np.uint64) + (np.uint64(seed) << np.uint64(40)) + _GOLDEN
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
        x = x ^ (x >> np.uint64(31))
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


def uniform(count, seed, offset=0, chunk=1 << 24, out=None):
    """z[0:count] for global indices offset .. offset+count-1."""
    if out is None:
        out = np.empty(count, dtype=np.float64)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        out[s:e] = uniform_from_index(np.arange(offset + s, offset + e, dtype=np.uint64), seed)
    return out


def uniform_cells(cells, n3, seed, ncells_global=None):
    """z blocks for an explicit list of global cell indices (shape (len(cells), n3))."""
    cells = np.asarray(cells, dtype=np.uint64)
    g = cells[:, None] * np.uint64(n3) + np.arange(n3, dtype=np.uint64)[None, :]
    return uniform_from_index(g, seed)


# ---- Problem A coefficient field (NEXT-1; tensor-valued, constant per cell)
# Per cell e (GLOBAL cell index), six uniforms u_i = U(seed, 6 e + i) give a symmetric,
# strictly diagonally dominant (hence SPD) tensor
#     D00, D11, D22 = 1.5 + 0.5 u_0..2  in [1, 2],   D01, D02, D12 = 0.25 u_3..5  in [-1/4, 1/4].
# Scales are powers of two, so every entry is the same double on the host (numpy) and on
# the device (torch ops on dg_fill_uniform_cells output): partition- and device-independent.
def tensor_field_from_uniforms(u6):
    """[ncell, 6] uniforms -> [ncell, 9] row-major tensors (numpy or torch arrays)."""
    d = 1.5 + 0.5 * u6[:, 0:3]
    o = 0.25 * u6[:, 3:6]
    cols = [d[:, 0], o[:, 0], o[:, 1], o[:, 0], d[:, 1], o[:, 2], o[:, 1], o[:, 2], d[:, 2]]
    if isinstance(u6, np.ndarray):
        return np.stack(cols, axis=1)
    import torch
    return torch.stack(cols, dim=1).contiguous()


def tensor_field_cells(cells, seed):
    """Host tensors [len(cells), 9] of the Problem A field for explicit global cell indices."""
    return tensor_field_from_uniforms(uniform_cells(cells, 6, seed))


# ---- multilinear meshes (NEXT-3: Problem C's "multilinear geometries") -------
# The paper does not print its meshes. The stand-in: the box's regular vertex grid with every
# vertex moved by amp * h_q * U(seed, 3 g + q) in each direction q (g = the GLOBAL vertex index
# ix + (Nx+1)(iy + (Ny+1) iz)); vertices on a Dirichlet side of the box keep their normal
# coordinate (the domain stays the box); along a periodic direction the perturbation of vertex
# N_q is that of vertex 0 (the grid stays periodic). With amp < 1/6 every edge vector of a cell
# has its own-direction component >= (1 - 2 amp) h and the other two <= 2 amp h, so every
# Jacobian (a convex combination of edge vectors per column) is column diagonally dominant with
# a positive diagonal: det J > 0 everywhere. Larger amp is allowed but not guaranteed valid
# (dg_set_geometry checks det J > 0 at every quadrature point and corner).
def vertex_grid(ncells, lo, hi, amp, seed, periodic=(0, 0, 0), box=None):
    """Vertex coordinates [iz][iy][ix][3] of the global grid (or of the sub-box
    box = ((i0, j0, k0), (i1, j1, k1)) of vertex indices, i1 exclusive; indices outside
    0..N are wrapped on periodic directions, clamped otherwise)."""
    N = [int(v) for v in ncells]
    h = [(hi[q] - lo[q]) / N[q] for q in range(3)]
    if box is None:
        box = ((0, 0, 0), (N[0] + 1, N[1] + 1, N[2] + 1))
    (i0, j0, k0), (i1, j1, k1) = box
    ks, js, is_ = np.arange(k0, k1), np.arange(j0, j1), np.arange(i0, i1)
    K, Jg, I = np.meshgrid(ks, js, is_, indexing="ij")
    idx = [I, Jg, K]
    out = np.empty(K.shape + (3,))
    for q in range(3):
        v = idx[q]
        if periodic[q]:
            shift = np.floor_divide(v, N[q])            # whole periods (a vertex index beyond the box)
            base = np.mod(v, N[q])
        else:
            shift = np.zeros_like(v)
            base = np.clip(v, 0, N[q])
        out[..., q] = lo[q] + (base + shift * N[q]) * h[q]
        if not periodic[q] and np.any((v < 0) | (v > N[q])):
            out[..., q] += (v - base) * h[q]             # regular continuation outside a Dirichlet box
    # perturbation by the wrapped vertex index
    wr = []
    for q in range(3):
        v = idx[q]
        wr.append(np.mod(v, N[q]) if periodic[q] else np.clip(v, 0, N[q]))
    g = (wr[0] + (N[0] + 1) * (wr[1] + (N[1] + 1) * wr[2])).astype(np.uint64)
    for q in range(3):
        d = amp * h[q] * uniform_from_index(3 * g + np.uint64(q), seed)
        if not periodic[q]:
            d = np.where((wr[q] == 0) | (wr[q] == N[q]), 0.0, d)   # the box sides stay planar
        out[..., q] += d
    return out
