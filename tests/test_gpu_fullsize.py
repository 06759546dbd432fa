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


@pytest.mark.parametrize("k", [2, 5, 7, 8])   # register (n = 3), 3-cell CTAs (n = 6), TMA (n = 8), bulk (n = 9)
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


@pytest.mark.parametrize("k", [2, 3])
def test_problem_c_full_size_sampled_vs_geometry_oracle(k):
    """The Problem C stand-in at its full size (~4e8 DOFs: multilinear periodic mesh, q = 3p+4;
    the bench's workload c-kK, through dg.from_config as bench.py runs it) against the geometry
    oracle O-2g on the 3 x 3 x 3-cell sub-mesh around sampled cells: the sub-mesh's vertices are
    the full mesh's (inputs.vertex_grid over that vertex box), its middle cell has all six
    neighbours inside it, so O-2g's y there is the full mesh's."""
    from oracle import o2_geometry as o2g
    from paper_1711_10885_b200 import dg
    cfg = configs.problem_c(k)
    op = dg.from_config(cfg)
    z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
    op.fill_uniform_local(z, cfg.seed)
    y = torch.empty_like(z)
    op.apply(z, y)
    torch.cuda.synchronize()
    N = cfg.ncells
    n3 = cfg.n3
    ymax = float(y.abs().max())
    rng = np.random.default_rng(7 + k)
    picks = [(0, 0, 0), (N[0] - 1, N[1] // 2, N[2] - 1)] + [tuple(int(v) for v in rng.integers(0, N[0], 3))
                                                          for _ in range(3)]
    worst = 0.0
    for c in picks:
        # the sub-mesh's cells (periodic wrap of the global indices) and vertex box
        idx = [[(c[q] + d) % N[q] for d in (-1, 0, 1)] for q in range(3)]
        cells = np.array([idx[0][a] + N[0] * (idx[1][b] + N[1] * idx[2][cc])
                          for cc in range(3) for b in range(3) for a in range(3)])
        box = (tuple(c[q] - 1 for q in range(3)), tuple(c[q] + 3 for q in range(3)))
        X = inputs.vertex_grid(cfg.ncells, cfg.lo, cfg.hi, cfg.geo_amp, cfg.geo_seed, cfg.periodic, box=box)
        zsub = inputs.uniform_cells(cells, n3, cfg.seed).reshape(-1)
        A = o2g.assemble((3, 3, 3), X, k, cfg.D, cfg.b, cfg.c, cfg.sigma, m=cfg.m)
        ysub = (A @ zsub).reshape(27, n3)[13]
        mid = cells[13]
        yg = y[mid * n3:(mid + 1) * n3].cpu().numpy()
        worst = max(worst, float(np.abs(yg - ysub).max()))
    op.close()
    assert worst <= TOL * ymax, (worst, ymax)
