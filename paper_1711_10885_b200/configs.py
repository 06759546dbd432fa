"""The five BASELINE.json configurations as data (mesh, degree, coefficients,
penalty, seed). No method arithmetic. Readings C-10, C-11, C-12, C-20 of
DESIGN.md fix what BASELINE.json leaves open (all-Dirichlet boundaries,
sigma = 3k(k+2)/h_min, the weak-scaling domain, the C4 meshes)."""
from dataclasses import dataclass, field
from typing import Tuple

import numpy as np


@dataclass
class Config:
    name: str
    ncells: Tuple[int, int, int]
    lo: Tuple[float, float, float]
    hi: Tuple[float, float, float]
    k: int
    D: Tuple[float, ...]
    b: Tuple[float, float, float]
    c: float
    sigma: float
    seed: int
    parts: Tuple[int, int, int] = (1, 1, 1)
    periodic: Tuple[int, int, int] = (0, 0, 0)
    dfield_seed: int = -1          # >= 0: per-cell tensor field inputs.tensor_field_* (Problem A)
    bkind: int = 0                 # velocity field: 0 constant b, 1 Taylor-Green (NEXT-2)
    m: int = 0                     # Gauss points per direction (0: k+1)
    geo_amp: float = 0.0           # > 0: multilinear mesh, inputs.vertex_grid(..., geo_amp, geo_seed) (NEXT-3)
    geo_seed: int = 0

    @property
    def n3(self):
        return (self.k + 1) ** 3

    @property
    def ncell(self):
        return self.ncells[0] * self.ncells[1] * self.ncells[2]

    @property
    def ndofs(self):
        return self.ncell * self.n3

    @property
    def h(self):
        return tuple((self.hi[q] - self.lo[q]) / self.ncells[q] for q in range(3))

    def args(self):
        """Positional (ncells, lo, hi, k, D, b, c, sigma) as used by the oracle functions."""
        return (self.ncells, self.lo, self.hi, self.k, self.D, self.b, self.c, self.sigma)


I3 = (1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0)
B_A = (1.0, 0.5, 0.25)


def sigma_for(k, h_min):
    """sigma = 3 k (k+2) / h_min (BASELINE.json configs; alpha = 3, reading C-4/C-11)."""
    return 3.0 * k * (k + 2) / h_min


def c1():
    return Config("C1", (4, 4, 4), (0, 0, 0), (1, 1, 1), 2, I3, B_A, 1.0, sigma_for(2, 0.25), 0)


def c2():
    D = (1.0, 0, 0, 0, 2.0, 0, 0, 0, 0.5)
    return Config("C2", (32, 32, 32), (0, 0, 0), (1, 1, 1), 3, D, (1.0, -1.0, 0.5), 0.1,
                  sigma_for(3, 1.0 / 32), 1)


def c3():
    return Config("C3", (128, 64, 64), (0, 0, 0), (2, 1, 1), 7, I3, B_A, 1.0, sigma_for(7, 1.0 / 64), 2)


def c4(k):
    N = int(round(464.16 / (k + 1)))
    return Config("C4-k%d" % k, (N, N, N), (0, 0, 0), (1, 1, 1), k, I3, B_A, 1.0, sigma_for(k, 1.0 / N), 3)


def c5_strong(parts=(1, 1, 1)):
    return Config("C5-strong", (256, 128, 128), (0, 0, 0), (1, 1, 1), 7, I3, B_A, 1.0,
                  sigma_for(7, 1.0 / 256), 4, parts)


_WEAK_GRID = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}


def c5_weak(P=1):
    """128x128x64 cells per GPU at h = 1/128 (reading C-12)."""
    px, py, pz = _WEAK_GRID[P]
    nc = (128 * px, 128 * py, 64 * pz)
    return Config("C5-weak-P%d" % P, nc, (0, 0, 0), tuple(v / 128.0 for v in nc), 7, I3, B_A, 1.0,
                  sigma_for(7, 1.0 / 128), 4, (px, py, pz))


def c3_weak(P=1):
    """C3's per-GPU block (128x64x64 cells, h = 1/64, k = 7) replicated over a Px x Py x Pz grid."""
    px, py, pz = _WEAK_GRID[P]
    nc = (128 * px, 64 * py, 64 * pz)
    return Config("C3-weak-P%d" % P, nc, (0, 0, 0), tuple(v / 64.0 for v in nc), 7, I3, B_A, 1.0,
                  sigma_for(7, 1.0 / 64), 2, (px, py, pz))


def problem_a(k, P=1):
    """The paper's Problem A (Table 1 protocol :933-936) as a synthetic stand-in:
    periodic in every direction, axis-parallel unit-box mesh of N^3 cubes with N = round(736.8/(k+1))
    so the DOF count is ~4e8 (3.2 GB vectors), q = 2p (n = m = k+1), a per-cell SPD tensor field
    (inputs.tensor_field_*, seed 6), b = (1, 1/2, 1/4), c = 1, sigma = 3k(k+2)N (as C-20).
    P > 1: the same block per GPU on a Px x Py x Pz grid (weak scaling)."""
    N = int(round(736.8 / (k + 1)))
    px, py, pz = _WEAK_GRID[P]
    nc = (N * px, N * py, N * pz)
    return Config("A-k%d" % k if P == 1 else "A-k%d-P%d" % (k, P), nc, (0, 0, 0), (float(px), float(py), float(pz)),
                  k, I3, B_A, 1.0, sigma_for(k, 1.0 / N), 5, (px, py, pz), (1, 1, 1), 6)


def problem_a_matrix(k, budget_bytes=24e9):
    """Problem A (as problem_a) on the mesh the matrix-based comparison can hold (NEXT-4; the paper
    also scales its matrix-based runs down): N^3 cells with the assembled
    block-stencil matrix (7 n^6 doubles per cell, include/dg.h) within budget_bytes, N >= 3 and a
    multiple of 3."""
    n = k + 1
    N = max(3, int((budget_bytes / (56.0 * n ** 6)) ** (1.0 / 3.0)))
    N -= N % 3          # 27 colour classes for dg_assemble's probes (a periodic tail adds classes)
    return Config("MB-k%d" % k, (N, N, N), (0, 0, 0), (1.0, 1.0, 1.0), k, I3, B_A, 1.0, sigma_for(k, 1.0 / N), 5,
                  (1, 1, 1), (1, 1, 1), 6)


def taylor_green(k, N=None):
    """The paper's transport run as an operator workload: the periodic box
    (-pi, pi)^3, D = 5e-6 I, c = 0, the Taylor-Green field b(x) (eq:2) at every quadrature point,
    q = 2p + 4 (m = k + 3). N^3 cells with N = round(736.8 / (k+1)) (~4e8 DOFs) by default; the
    paper's production mesh is N = 240 at k = 5. sigma = 3k(k+2)/h."""
    if N is None:
        N = int(round(736.8 / (k + 1)))
    h = 2 * np.pi / N
    d = 5e-6
    return Config("TG-k%d" % k, (N, N, N), (-np.pi,) * 3, (np.pi,) * 3, k, (d, 0, 0, 0, d, 0, 0, 0, d), (0.0, 0.0, 0.0),
                  0.0, sigma_for(k, h), 8, (1, 1, 1), (1, 1, 1), -1, 1, k + 3)


D_C = (1.0, 0.25, 0.125, 0.25, 1.5, -0.25, 0.125, -0.25, 0.75)   # a fixed full SPD tensor


def problem_c(k, P=1, m=None):
    """The paper's Problem C as a synthetic stand-in: "multilinear geometries" --
    the periodic unit box's N^3 grid with every vertex moved by up to 0.15 h per direction
    (inputs.vertex_grid, seed 9; below 1/6 every Jacobian is column diagonally dominant, so no
    cell of the ~1e6-5e7 can invert), N = round(736.8/(k+1)) (~4e8 DOFs, the Table 1 protocol
    PAPER.md:933-936) -- and q = 3p + 4, i.e. m = ceil((3k+5)/2) Gauss points per direction (m <= 16;
    k = 10 falls back to m = 13). The paper's polynomial coefficients are not printed: a constant
    full SPD tensor D_C, b = (1, 1/2, 1/4), c = 1, sigma = 3k(k+2)N. P > 1: the same block per GPU."""
    N = int(round(736.8 / (k + 1)))
    if m is None:
        m = -(-(3 * k + 5) // 2)
        if m > 16:
            m = k + 3
    px, py, pz = _WEAK_GRID[P]
    nc = (N * px, N * py, N * pz)
    return Config("C-k%d" % k if P == 1 else "C-k%d-P%d" % (k, P), nc, (0, 0, 0), (float(px), float(py), float(pz)),
                  k, D_C, B_A, 1.0, sigma_for(k, 1.0 / N), 10, (px, py, pz), (1, 1, 1), -1, 0, m, 0.15, 9)


def by_name(name):
    name = name.lower()
    table = {"c1": c1, "c2": c2, "c3": c3, "c5strong": c5_strong, "c5weak": c5_weak}
    if name.startswith("c4-k"):
        return c4(int(name[4:]))
    if name.startswith("a-k"):
        return problem_a(int(name[3:]))
    if name.startswith("tg-k"):
        return taylor_green(int(name[4:]))
    if name.startswith("mb-k"):
        return problem_a_matrix(int(name[4:]))
    if name.startswith("c-k"):
        return problem_c(int(name[3:]))
    return table[name]()


def small(k, ncells=(3, 2, 2), lo=(0, 0, 0), hi=(1.5, 1.0, 0.5), D=(1, 0, 0, 0, 2, 0, 0, 0, 0.5),
          b=(1.0, -0.5, 0.25), c=0.3, seed=7):
    """Survey test mesh (SURVEY.md 8(c) 'Verification'): anisotropic cells."""
    h = [(hi[q] - lo[q]) / ncells[q] for q in range(3)]
    return Config("small-k%d" % k, tuple(ncells), tuple(lo), tuple(hi), k, tuple(float(v) for v in D),
                  tuple(b), c, sigma_for(k, min(h)), seed)
