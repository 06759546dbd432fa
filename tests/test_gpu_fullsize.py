"""Parity at the BASELINE.json full sizes, in the launch configuration bench.py times.

The oracle cannot run a 1e8..2e9-DOF mesh, so each check takes one z-layer of cells: the
layer and its two z-neighbour layers are copied to the host and O-1 is run on that 3-layer
sub-mesh (same cell size h, same sigma; its box is the slab [z0-1, z0+2) h). Every cell of
the middle layer has all of its neighbours inside the sub-mesh, and the x/y box sides are
the real ones, so O-1's y on the middle layer is the full mesh's y there (the sub-mesh's
own z-sides only touch the outer layers, which are not compared). Compared: a seeded
sample of middle-layer cells incl. the layer's corners and edges, elementwise at
1e-12 * max|y| (reading C-14), where max|y| is the full vector's.
"""
import numpy as np
import pytest

from oracle import o1
from paper_1711_10885_b200 import configs, inputs

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def slab_check(cfg, z, y, z0, count, seed, Dcell_fn=None):
    """Compare the GPU y on z-layer z0 with O-1 on the 3-layer sub-mesh around it."""
    nx, ny, nz = cfg.ncells
    n3 = cfg.n3
    per_layer = nx * ny
    lay = [((z0 + d) % nz) for d in (-1, 0, 1)]
    if not cfg.periodic[2]:
        assert 1 <= z0 <= nz - 2
    zs = np.concatenate([z[l * per_layer * n3:(l + 1) * per_layer * n3].cpu().numpy() for l in lay])
    ymid = y[z0 * per_layer * n3:(z0 + 1) * per_layer * n3].cpu().numpy().reshape(per_layer, n3)
    h = cfg.h
    lo = (cfg.lo[0], cfg.lo[1], cfg.lo[2] + (z0 - 1) * h[2])
    hi = (cfg.hi[0], cfg.hi[1], cfg.lo[2] + (z0 + 2) * h[2])
    rng = np.random.default_rng(seed)
    edge = [x + nx * yy for x in (0, nx // 2, nx - 1) for yy in (0, ny // 2, ny - 1)]
    cells2d = np.unique(np.r_[edge, rng.integers(0, per_layer, count)]).astype(np.int64)
    kw = {"periodic": (cfg.periodic[0], cfg.periodic[1], 0)}
    if Dcell_fn is not None:
        glob = np.concatenate([np.arange(per_layer) + l * per_layer for l in lay])
        kw["Dcell"] = Dcell_fn(glob)
    ys, _ = o1.apply((nx, ny, 3), lo, hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma, zs, cells=cells2d + per_layer, **kw)
    return np.abs(ymid[cells2d] - ys).max()


def run_full(cfg, general=False):
    from paper_1711_10885_b200 import dg
    op = dg.from_config(cfg)
    if general:
        op.set_tensor_field(cfg.dfield_seed)
    z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
    op.fill_uniform_local(z, cfg.seed)
    y = torch.full_like(z, float("nan"))
    op.apply(z, y)
    torch.cuda.synchronize()
    op.close()
    return z, y


@pytest.mark.parametrize("k", list(range(1, 11)))
def test_c4_full_size_slab(k):
    cfg = configs.c4(k)
    z, y = run_full(cfg)
    ymax = float(y.abs().max())
    assert np.isfinite(ymax)
    for z0, seed in ((1, 0), (cfg.ncells[2] // 2, 1), (cfg.ncells[2] - 2, 2)):
        assert slab_check(cfg, z, y, z0, 150, seed) <= TOL * ymax
    del z, y
    torch.cuda.empty_cache()


def test_c5_strong_max_size_slab():
    """2^31 DOFs (17.2 GB per vector) on one GPU: the 64-bit offsets of the ABI and kernel."""
    cfg = configs.c5_strong()
    assert cfg.ndofs == 2 ** 31
    z, y = run_full(cfg)
    ymax = float(y.abs().max())
    assert np.isfinite(ymax) and not bool(torch.isnan(y).any())
    for z0, seed in ((1, 0), (cfg.ncells[2] - 2, 1)):
        assert slab_check(cfg, z, y, z0, 120, seed) <= TOL * ymax
    del z, y
    torch.cuda.empty_cache()


def test_c5_weak_block_slab():
    cfg = configs.c5_weak(1)
    z, y = run_full(cfg)
    ymax = float(y.abs().max())
    for z0, seed in ((1, 3), (cfg.ncells[2] // 2, 4), (cfg.ncells[2] - 2, 5)):
        assert slab_check(cfg, z, y, z0, 120, seed) <= TOL * ymax
    del z, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", [2, 7])
def test_problem_a_full_size_slab(k):
    """The paper's Problem A at ~4e8 DOFs (periodic, per-cell tensor field) on the general kernel;
    the slab wraps around the periodic z sides."""
    cfg = configs.problem_a(k)
    z, y = run_full(cfg, general=True)
    ymax = float(y.abs().max())
    assert np.isfinite(ymax)
    for z0, seed in ((0, 0), (cfg.ncells[2] - 1, 1), (cfg.ncells[2] // 3, 2)):
        err = slab_check(cfg, z, y, z0, 100, seed,
                         Dcell_fn=lambda glob: inputs.tensor_field_cells(glob, cfg.dfield_seed))
        assert err <= TOL * ymax
    del z, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", list(range(1, 11)))
def test_c4_full_vector_vs_o3(k):
    """Every element of the C4 vectors (~1e8 DOFs) against the Kronecker closed form O-3 (SURVEY.md 4:
    "O-3: full on every config")."""
    from oracle import o3_kron as o3
    cfg = configs.c4(k)
    z, y = run_full(cfg)
    zn = z.cpu().numpy()
    yn = y.cpu().numpy()
    del z, y
    torch.cuda.empty_cache()
    y3 = o3.apply(*cfg.args(), zn)
    assert np.abs(yn - y3).max() <= TOL * np.abs(y3).max()
