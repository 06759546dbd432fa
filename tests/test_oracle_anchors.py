"""The oracle against the independent survey computation (SURVEY.md 8(c)
'Parity anchors'), which fixes the seeded RNG (reading C-13) and every
convention C-2..C-13 in executable form. Elementwise anchors at 1e-12 * max|y|,
sums and norms at 1e-10 relative."""
import numpy as np
import pytest

from conftest import golden
from oracle import o1, o3_kron as o3
from paper_1711_10885_b200 import configs, inputs


def check(y, a):
    N = y.size
    s = a["max_abs"]
    assert abs(np.abs(y).max() - s) <= 1e-12 * s
    for key, idx in (("y0", 0), ("y1", 1), ("yhalf", N // 2), ("ylast", N - 1)):
        if key in a:
            assert abs(y[idx] - a[key]) <= 1e-12 * s, key
    if "sum" in a:
        assert abs(y.sum() - a["sum"]) <= 1e-10 * abs(a["sum"])
    assert abs(np.linalg.norm(y) - a["norm2"]) <= 1e-10 * a["norm2"]


def test_rng_anchor():
    g = golden("anchors.json")["rng"]
    z = inputs.uniform(2, g["seed"])
    assert z[0] == g["z0"] and z[1] == g["z1"]


def test_c1_anchor_o1_o3():
    cfg = configs.c1()
    z = inputs.uniform(cfg.ndofs, cfg.seed)
    a = golden("anchors.json")["C1"]
    y1, _ = o1.apply(*cfg.args(), z)
    check(y1, a)
    check(o3.apply(*cfg.args(), z), a)


@pytest.mark.parametrize("which", ["C1_mass_only", "C1_convection_only", "C1_diffusion_only"])
def test_c1_isolated_coefficients(which):
    g = golden("anchors.json")
    a = g[which]
    cfg = configs.c1()
    z = inputs.uniform(cfg.ndofs, cfg.seed)
    args = (cfg.ncells, cfg.lo, cfg.hi, cfg.k, a["D"], a["b"], a["c"], g["C1_isolated_sigma"])
    y1, _ = o1.apply(*args, z)
    check(y1, a)
    assert abs(z @ y1 - a["zTy"]) <= 1e-12 * abs(a["zTy"])


def test_c2_anchor_o3_and_sampled_o1():
    cfg = configs.c2()
    z = inputs.uniform(cfg.ndofs, cfg.seed)
    a = golden("anchors.json")["C2"]
    y3 = o3.apply(*cfg.args(), z)
    check(y3, a)
    rng = np.random.default_rng(0)
    cells = np.unique(np.r_[0, cfg.ncell - 1, rng.integers(0, cfg.ncell, 40)])
    ys, _ = o1.apply(*cfg.args(), z, cells=cells)
    n3 = cfg.n3
    ref = y3.reshape(-1, n3)[cells]
    assert np.abs(ys - ref).max() <= 1e-12 * a["max_abs"]
