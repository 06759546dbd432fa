"""CUDA path (through the C ABI) against the oracle, element by element, on the
same seeded inputs. Tolerance: max|y - y_ref| <= 1e-12 max|y_ref| (BASELINE.json
north_star; metric reading C-14). Sizes span several CTAs and ragged tails; full
BASELINE sizes are checked on sampled cells (O-1 sampled mode) and by the anchors.
"""
import numpy as np
import pytest

from conftest import golden
from oracle import o1, o3_kron as o3, rhs
from paper_1711_10885_b200 import configs, inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12


def dgmod():
    from paper_1711_10885_b200 import dg
    return dg


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def gpu_apply(cfg, z_np, terms=7, D=None, b=None, c=None, sigma=None):
    dg = dgmod()
    op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D if D is None else D, cfg.b if b is None else b,
                     cfg.c if c is None else c, cfg.sigma if sigma is None else sigma)
    z = torch.from_numpy(z_np).cuda()
    y = torch.full_like(z, float("nan"))
    op.apply(z, y, terms=terms)
    torch.cuda.synchronize()
    op.close()
    return y.cpu().numpy()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dgmod().lib()


@pytest.mark.parametrize("mask", [1, 2, 4, 3, 5, 6, 7])
def test_c1_masks_vs_o1(mask):
    cfg = configs.c1()
    z = inputs.uniform(cfg.ndofs, cfg.seed)
    y = gpu_apply(cfg, z, terms=mask)
    yref, _ = o1.apply(*cfg.args(), z, mask=mask)
    assert rel(y, yref) < TOL


def test_c1_anchor():
    cfg = configs.c1()
    z = inputs.uniform(cfg.ndofs, cfg.seed)
    y = gpu_apply(cfg, z)
    a = golden("anchors.json")["C1"]
    assert abs(y[0] - a["y0"]) <= TOL * a["max_abs"] and abs(y[-1] - a["ylast"]) <= TOL * a["max_abs"]
    assert abs(np.linalg.norm(y) - a["norm2"]) <= 1e-10 * a["norm2"]


@pytest.mark.parametrize("k", list(range(1, 11)))
def test_every_degree_vs_o1(k):
    """Anisotropic cells, negative velocity component, ragged CTA tail (ncell not a multiple of C)."""
    cfg = configs.small(k, ncells=(5, 3, 2), lo=(0.1, -0.2, 0.0), hi=(1.6, 0.7, 0.5), b=(1.0, -0.5, 0.25), c=0.3)
    z = inputs.uniform(cfg.ndofs, 100 + k)
    y = gpu_apply(cfg, z)
    yref, _ = o1.apply(*cfg.args(), z)
    assert rel(y, yref) < TOL


@pytest.mark.parametrize("k", [1, 2, 3, 7, 10])
@pytest.mark.parametrize("ncells", [(1, 1, 1), (1, 1, 4), (7, 1, 1), (2, 3, 1)])
def test_degenerate_meshes(k, ncells):
    cfg = configs.small(k, ncells=ncells, hi=(1.0, 0.5, 2.0))
    z = inputs.uniform(cfg.ndofs, 9)
    y = gpu_apply(cfg, z)
    yref, _ = o1.apply(*cfg.args(), z)
    assert rel(y, yref) < TOL


@pytest.mark.parametrize("which", ["mass", "convection", "diffusion"])
@pytest.mark.parametrize("k", [2, 7])
def test_isolated_coefficients(which, k):
    """small terms are invisible at 1e-12 of the full operator, so each
    coefficient is checked on its own, per mask."""
    D, b, c = {"mass": ((0,) * 9, (0, 0, 0), 1.0), "convection": ((0,) * 9, (1.0, -0.5, 0.25), 0.0),
               "diffusion": ((1, 0, 0, 0, 2, 0, 0, 0, 0.5), (0, 0, 0), 0.0)}[which]
    cfg = configs.small(k, ncells=(4, 3, 3), D=D, b=b, c=c)
    z = inputs.uniform(cfg.ndofs, 5)
    for mask in (1, 2, 4, 7):
        y = gpu_apply(cfg, z, terms=mask)
        yref, _ = o1.apply(*cfg.args(), z, mask=mask)
        if np.abs(yref).max() == 0:
            assert np.abs(y).max() == 0
        else:
            assert rel(y, yref) < TOL


def test_mass_invariant_exact():
    cfg = configs.small(5, D=(0,) * 9, b=(0, 0, 0), c=0.7)
    z = inputs.uniform(cfg.ndofs, 4)
    y = gpu_apply(cfg, z)
    assert np.all(np.isfinite(y))
    assert rel(y, 0.7 * np.prod(cfg.h) * z) < 1e-14


def test_symmetry_b0():
    cfg = configs.small(4, ncells=(3, 3, 2), b=(0, 0, 0))
    z = inputs.uniform(cfg.ndofs, 1)
    w = inputs.uniform(cfg.ndofs, 2)
    yz = gpu_apply(cfg, z)
    yw = gpu_apply(cfg, w)
    assert abs(w @ yz - z @ yw) < 1e-13 * abs(w @ yz)


def test_upwind_energy_identity():
    cfg = configs.c1()
    z = inputs.uniform(cfg.ndofs, 0)
    y = gpu_apply(cfg, z, D=(0,) * 9, c=0.0)
    E = rhs.upwind_energy(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.b, z)
    assert abs(z @ y - E) < 1e-12 * E


@pytest.mark.parametrize("k", [1, 3, 6, 7])
def test_residual_polynomial_consistency(k):
    """dg_residual(z*, F) ~ 0 for u* in Q_k (reading C-1)."""
    dg = dgmod()
    cfg = configs.small(k, ncells=(3, 2, 2))
    zs, F = rhs.consistency_data(*cfg.args(), seed=k)
    op = dg.from_config(cfg)
    zt = torch.from_numpy(zs).cuda()
    ft = torch.from_numpy(F).cuda()
    r = torch.empty_like(zt)
    op.residual(zt, ft, r)
    torch.cuda.synchronize()
    assert np.abs(r.cpu().numpy()).max() < 1e-12 * np.abs(F).max()
    # and the residual epilogue is exactly f - (A z) of the apply path
    y = torch.empty_like(zt)
    op.apply(zt, y)
    torch.cuda.synchronize()
    assert np.array_equal(r.cpu().numpy(), (ft - y).cpu().numpy())
    op.close()


def test_device_rng_matches_numpy():
    dg = dgmod()
    t = torch.empty(100_003, dtype=torch.float64, device="cuda")
    dg.fill_uniform(t, 5, offset=12345)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), inputs.uniform(100_003, 5, offset=12345))


def test_c2_full_vs_o3_and_anchor():
    dg = dgmod()
    cfg = configs.c2()
    op = dg.from_config(cfg)
    z = torch.empty(cfg.ndofs, dtype=torch.float64, device="cuda")
    op.fill_uniform_local(z, cfg.seed)
    y = torch.empty_like(z)
    op.apply(z, y)
    torch.cuda.synchronize()
    zn = inputs.uniform(cfg.ndofs, cfg.seed)
    assert np.array_equal(z.cpu().numpy(), zn)
    yn = y.cpu().numpy()
    y3 = o3.apply(*cfg.args(), zn)
    assert rel(yn, y3) < TOL
    a = golden("anchors.json")["C2"]
    assert abs(yn[0] - a["y0"]) <= TOL * a["max_abs"]
    assert abs(yn[-1] - a["ylast"]) <= TOL * a["max_abs"]
    assert abs(yn.sum() - a["sum"]) <= 1e-10 * abs(a["sum"])
    op.close()


def sampled_cells(cfg, count, seed):
    """Random cells plus every boundary type: the 8 corners and a cell on each face/edge."""
    rng = np.random.default_rng(seed)
    nx, ny, nz = cfg.ncells
    special = []
    for x in (0, nx // 2, nx - 1):
        for y in (0, ny // 2, ny - 1):
            for z in (0, nz // 2, nz - 1):
                special.append(x + nx * (y + ny * z))
    return np.unique(np.r_[special, rng.integers(0, cfg.ncell, count)]).astype(np.int64)


@pytest.mark.slow
def test_c3_full_size_sampled_vs_o1():
    """BASELINE config 3 at full size (268M DOFs) in the bench's launch configuration."""
    dg = dgmod()
    cfg = configs.c3()
    op = dg.from_config(cfg)
    z = torch.empty(cfg.ndofs, dtype=torch.float64, device="cuda")
    op.fill_uniform_local(z, cfg.seed)
    y = torch.empty_like(z)
    op.apply(z, y)
    torch.cuda.synchronize()
    zn = z.cpu().numpy()
    yn = y.cpu().numpy()
    del z, y
    op.close()
    cells = sampled_cells(cfg, 300, 0)
    ys, _ = o1.apply(*cfg.args(), zn, cells=cells)
    got = yn.reshape(-1, cfg.n3)[cells]
    a = golden("anchors.json")["C3"]
    assert np.abs(got - ys).max() <= TOL * a["max_abs"]
    assert abs(np.abs(yn).max() - a["max_abs"]) <= TOL * a["max_abs"]
    for key, idx in (("y0", 0), ("y1", 1), ("yhalf", yn.size // 2), ("ylast", yn.size - 1)):
        assert abs(yn[idx] - a[key]) <= TOL * a["max_abs"], key
    assert abs(np.linalg.norm(yn) - a["norm2"]) <= 1e-10 * a["norm2"]
