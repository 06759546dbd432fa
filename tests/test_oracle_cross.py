"""O-1 (naive C) == O-2 (assembled from the weak form) == O-3 (Kronecker closed
form), per term mask, on small anisotropic meshes."""
import numpy as np
import pytest

from oracle import o1, o2_assembled as o2, o3_kron as o3
from paper_1711_10885_b200 import configs, inputs


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def spd(seed):
    rng = np.random.default_rng(seed)
    M = rng.normal(size=(3, 3))
    return tuple((M @ M.T + 0.5 * np.eye(3)).ravel())


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("mask", [1, 2, 4, 7])
def test_o1_o2_o3_diag(k, mask):
    cfg = configs.small(k)
    z = inputs.uniform(cfg.ndofs, 11 + k)
    y1, _ = o1.apply(*cfg.args(), z, mask=mask)
    A = o2.assemble(*cfg.args(), mask=mask)
    y3 = o3.apply(*cfg.args(), z, mask=mask)
    assert rel(y1, A @ z) < 1e-13
    assert rel(y3, A @ z) < 1e-13


@pytest.mark.parametrize("k", [1, 2])
def test_o1_o2_full_D_negative_b(k):
    cfg = configs.small(k, D=spd(k), b=(-0.7, 0.4, -1.1), c=0.7)
    z = inputs.uniform(cfg.ndofs, 3)
    y1, _ = o1.apply(*cfg.args(), z)
    A = o2.assemble(*cfg.args())
    assert rel(y1, A @ z) < 1e-13


def test_o1_o3_larger_mesh():
    cfg = configs.small(4, ncells=(5, 4, 3), hi=(1.0, 2.0, 0.75), b=(0.3, -1.0, 2.0))
    z = inputs.uniform(cfg.ndofs, 9)
    y1, _ = o1.apply(*cfg.args(), z)
    y3 = o3.apply(*cfg.args(), z)
    assert rel(y1, y3) < 1e-13


def test_o1_sampled_mode_matches_full():
    cfg = configs.small(3, ncells=(4, 3, 3))
    z = inputs.uniform(cfg.ndofs, 1)
    yf, _ = o1.apply(*cfg.args(), z)
    cells = np.array([0, 5, 17, cfg.ncell - 1])
    ys, _ = o1.apply(*cfg.args(), z, cells=cells)
    n3 = cfg.n3
    for i, e in enumerate(cells):
        assert np.array_equal(ys[i], yf[e * n3:(e + 1) * n3])


def test_o1_thread_count_independent():
    cfg = configs.small(2)
    z = inputs.uniform(cfg.ndofs, 2)
    ya, _ = o1.apply(*cfg.args(), z, nthreads=1)
    yb, _ = o1.apply(*cfg.args(), z, nthreads=4)
    assert np.array_equal(ya, yb)   # each cell is computed by one thread in a fixed order
