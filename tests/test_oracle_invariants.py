"""Invariants that pin the oracle to the paper rather than to itself
(SURVEY.md 8(c) P-3, P-4, P-10):
  * hand-derived one-cell matrices (golden/single_cell_k1.json)
  * mass matrix for D = 0, b = 0: A = c Delta_T I (orthonormal basis)
  * symmetry of the SIPG part for b = 0 (eq:blf)
  * polynomial consistency A z* = F (l_h; pins reading C-1)
  * upwind energy identity for D = 0, c = 0
  * upwind dependence: the convective face term reads only the upwind side
"""
import numpy as np
import pytest

from conftest import golden, num
from oracle import o1, o2_assembled as o2, o3_kron as o3, rhs
from paper_1711_10885_b200 import configs, inputs


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def test_single_cell_hand_cases():
    g = golden("single_cell_k1.json")
    m = g["mesh"]
    d = g["diffusion"]
    args = (m["ncells"], m["lo"], m["hi"], m["k"], d["D"], d["b"], d["c"], d["sigma"])
    A = o2.assemble(*args)
    assert np.abs(A - np.diag(d["diag"])).max() < 1e-12
    for j in range(8):
        e = np.zeros(8)
        e[j] = 1.0
        y1, _ = o1.apply(*args, e)
        assert np.abs(y1 - A[:, j]).max() < 1e-12
        assert np.abs(o3.apply(*args, e) - A[:, j]).max() < 1e-12
    cv = g["convection"]
    args = (m["ncells"], m["lo"], m["hi"], m["k"], cv["D"], cv["b"], cv["c"], cv["sigma"])
    e0 = np.zeros(8)
    e0[0] = 1.0
    want = np.array([num(v) for v in cv["column0"]])
    y1, _ = o1.apply(*args, e0)
    assert np.abs(y1 - want).max() < 1e-14
    assert np.abs(o2.assemble(*args)[:, 0] - want).max() < 1e-14


@pytest.mark.parametrize("k", [1, 2, 5])
def test_mass_invariant(k):
    cfg = configs.small(k, D=(0,) * 9, b=(0, 0, 0), c=0.7)
    z = inputs.uniform(cfg.ndofs, 4)
    y1, _ = o1.apply(*cfg.args(), z)
    dT = np.prod(cfg.h)
    assert np.all(np.isfinite(y1))
    assert rel(y1, 0.7 * dT * z) < 1e-14
    if k <= 2:
        A = o2.assemble(*cfg.args())
        assert np.abs(A - 0.7 * dT * np.eye(A.shape[0])).max() < 1e-14 * np.abs(A).max()


@pytest.mark.parametrize("full", [False, True])
def test_symmetry_without_convection(full):
    D = (1, 0, 0, 0, 2, 0, 0, 0, 0.5)
    if full:
        rng = np.random.default_rng(5)
        M = rng.normal(size=(3, 3))
        D = tuple((M @ M.T + 0.3 * np.eye(3)).ravel())
    cfg = configs.small(2, D=D, b=(0, 0, 0))
    A = o2.assemble(*cfg.args())
    assert np.abs(A - A.T).max() < 1e-13 * np.abs(A).max()
    # and the convective part alone is not symmetric (the test can fail)
    Ab = o2.assemble(*configs.small(2, D=(0,) * 9, c=0.0).args())
    assert np.abs(Ab - Ab.T).max() > 1e-3 * np.abs(Ab).max()
    # bilinear symmetry through O-1
    z = inputs.uniform(cfg.ndofs, 1)
    w = inputs.uniform(cfg.ndofs, 2)
    yz, _ = o1.apply(*cfg.args(), z)
    yw, _ = o1.apply(*cfg.args(), w)
    assert abs(w @ yz - z @ yw) < 1e-13 * abs(w @ yz)


@pytest.mark.parametrize("k,full", [(1, False), (2, False), (2, True), (3, False)])
def test_polynomial_consistency(k, full):
    D = (1, 0, 0, 0, 2, 0, 0, 0, 0.5)
    if full:
        rng = np.random.default_rng(8)
        M = rng.normal(size=(3, 3))
        D = tuple((M @ M.T + 0.3 * np.eye(3)).ravel())
    cfg = configs.small(k, D=D, b=(1.0, -0.5, 0.25), c=0.3)
    zs, F = rhs.consistency_data(*cfg.args(), seed=k)
    y1, _ = o1.apply(*cfg.args(), zs)
    assert rel(y1, F) < 1e-13
    A = o2.assemble(*cfg.args()) if k <= 2 else None
    if A is not None:
        assert rel(A @ zs, F) < 1e-13


@pytest.mark.parametrize("full", [False, True])
def test_consistency_separates_average_sign(full):
    """Reading C-1: PAPER.md:271 prints {v}_w = w- v- - w+ v+. With that sign the
    scheme is not consistent (residual O(1e-2)); with '+' it is (1e-15)."""
    D = (1, 0, 0, 0, 2, 0, 0, 0, 0.5)
    if full:
        rng = np.random.default_rng(8)
        M = rng.normal(size=(3, 3))
        D = tuple((M @ M.T + 0.3 * np.eye(3)).ravel())
    cfg = configs.small(2, D=D)
    zs, F = rhs.consistency_data(*cfg.args(), seed=1)
    assert rel(o2.assemble(*cfg.args()) @ zs, F) < 1e-13
    assert rel(o2.assemble(*cfg.args(), avg_sign=-1.0) @ zs, F) > 1e-3


def test_upwind_energy_identity():
    cfg = configs.c1()
    z = inputs.uniform(cfg.ndofs, 0)
    y, _ = o1.apply(cfg.ncells, cfg.lo, cfg.hi, cfg.k, (0,) * 9, cfg.b, 0.0, cfg.sigma, z)
    E = rhs.upwind_energy(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.b, z)
    assert abs(z @ y - E) < 1e-13 * E


def test_upwind_dependence():
    """For b_q > 0 the convective face term of the low cell reads only itself:
    perturbing the downwind neighbour leaves the D = 0 operator unchanged on the
    upwind cell in the convective-only problem for faces in +q direction."""
    cfg = configs.small(2, ncells=(2, 1, 1), D=(0,) * 9, b=(1.0, 0.0, 0.0), c=0.0)
    z = inputs.uniform(cfg.ndofs, 1)
    y, _ = o1.apply(*cfg.args(), z)
    z2 = z.copy()
    z2[cfg.n3:] += 1.0      # perturb downwind cell (x-high)
    y2, _ = o1.apply(*cfg.args(), z2)
    assert np.array_equal(y[:cfg.n3], y2[:cfg.n3])
    assert not np.allclose(y[cfg.n3:], y2[cfg.n3:])
