"""NEXT-1 on the GPU: periodic boundaries (fast kernel, constant diagonal D)
and the general-coefficient kernel (full symmetric D, per-cell tensors with live WSIPG
weights and harmonic penalty), each against the oracle O-1 element by element at the
north_star tolerance 1e-12 (max-norm relative, reading C-14)."""
import numpy as np
import pytest

from oracle import o1, o3_kron as o3
from paper_1711_10885_b200 import configs, inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1711_10885_b200 import dg
    dg.lib()


def run(cfg, z_np, periodic=(0, 0, 0), terms=7, Dcell=None):
    from paper_1711_10885_b200 import dg
    op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma,
                     bc=dg.bc_from_periodic(periodic))
    if Dcell is not None:
        op.set_diffusion(torch.from_numpy(np.ascontiguousarray(Dcell, dtype=np.float64).reshape(-1)).cuda())
    z = torch.from_numpy(z_np).cuda()
    y = torch.full_like(z, float("nan"))
    op.apply(z, y, terms=terms)
    torch.cuda.synchronize()
    op.close()
    return y.cpu().numpy()


def spd_field(ncell, seed, iso=0.5):
    rng = np.random.default_rng(seed)
    M = rng.normal(size=(ncell, 3, 3))
    return np.einsum("eij,ekj->eik", M, M) + iso * np.eye(3)[None]


PERIODIC = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1)]


@pytest.mark.parametrize("periodic", PERIODIC)
@pytest.mark.parametrize("k", [1, 2, 3, 5, 7, 8, 10])
def test_periodic_fast_kernel_vs_o1(k, periodic):
    cfg = configs.small(k, ncells=(5, 3, 2), lo=(0.1, -0.2, 0.0), hi=(1.6, 0.7, 0.5), b=(1.0, -0.5, 0.25), c=0.3)
    z = inputs.uniform(cfg.ndofs, 300 + k)
    for mask in (7, 2):
        y = run(cfg, z, periodic, terms=mask)
        yref, _ = o1.apply(*cfg.args(), z, mask=mask, periodic=periodic)
        assert rel(y, yref) < TOL


@pytest.mark.parametrize("k", [2, 7])
@pytest.mark.parametrize("ncells", [(1, 1, 1), (1, 2, 1), (2, 1, 3)])
def test_periodic_single_cell_directions(k, ncells):
    # a periodic direction with one cell: the cell is its own neighbour
    cfg = configs.small(k, ncells=ncells, hi=(0.5, 1.0, 0.75))
    z = inputs.uniform(cfg.ndofs, 17)
    y = run(cfg, z, (1, 1, 1))
    yref, _ = o1.apply(*cfg.args(), z, periodic=(1, 1, 1))
    assert rel(y, yref) < TOL


def test_periodic_c2_full_vs_o3():
    cfg = configs.c2()
    z = inputs.uniform(cfg.ndofs, cfg.seed)
    y = run(cfg, z, (1, 1, 1))
    y3 = o3.apply(*cfg.args(), z, periodic=(1, 1, 1))
    assert rel(y, y3) < TOL


def test_periodic_constant_state_is_mass():
    cfg = configs.small(7, ncells=(4, 4, 2), b=(1.0, -0.5, 0.25), c=0.45)
    z = np.zeros((cfg.ncell, cfg.n3))
    z[:, 0] = 1.3
    y = run(cfg, z.ravel(), (1, 1, 1))
    # A 1 = c Delta_T 1: the face terms cancel only up to rounding; they are larger than
    # max|y| by gamma |F| / (c |T|) ~ 756 * 0.0625 / 0.0105 ~ 4.5e3, hence 1e-11 (not 1e-16)
    assert rel(y, 0.45 * np.prod(cfg.h) * z.ravel()) < 1e-11


# ------------------------------------------------------------------ general-coefficient kernel

def full_D(seed):
    rng = np.random.default_rng(seed)
    M = rng.normal(size=(3, 3))
    return tuple((M @ M.T + 0.5 * np.eye(3)).ravel())


@pytest.mark.parametrize("k", list(range(1, 11)))
def test_full_constant_D_every_degree_vs_o1(k):
    cfg = configs.small(k, ncells=(5, 3, 2), lo=(0.1, -0.2, 0.0), hi=(1.6, 0.7, 0.5), D=full_D(k),
                        b=(1.0, -0.5, 0.25), c=0.3)
    z = inputs.uniform(cfg.ndofs, 400 + k)
    for mask in (1, 2, 4, 7):
        y = run(cfg, z, terms=mask)
        yref, _ = o1.apply(*cfg.args(), z, mask=mask)
        assert rel(y, yref) < TOL, mask


@pytest.mark.parametrize("periodic", [(0, 0, 0)] + PERIODIC)
@pytest.mark.parametrize("k", [1, 2, 4, 7, 10])
def test_percell_D_vs_o1(k, periodic):
    cfg = configs.small(k, ncells=(4, 3, 2), hi=(1.0, 0.75, 0.5), b=(-0.8, 0.4, 0.3), c=0.6)
    Dc = spd_field(cfg.ncell, 50 + k)
    z = inputs.uniform(cfg.ndofs, 500 + k)
    for mask in (1, 2, 4, 7):
        y = run(cfg, z, periodic, terms=mask, Dcell=Dc)
        yref, _ = o1.apply(*cfg.args(), z, mask=mask, periodic=periodic, Dcell=Dc)
        if np.abs(yref).max() == 0:
            assert np.abs(y).max() == 0
        else:
            assert rel(y, yref) < TOL, mask


@pytest.mark.parametrize("k", [2, 7])
def test_percell_diffusion_only_and_degenerate_D(k):
    # isolated diffusion + penalty, with some cells D = 0 (reading C-5: d- + d+ = 0)
    cfg = configs.small(k, ncells=(3, 3, 2), hi=(0.75, 0.75, 0.5), b=(0, 0, 0), c=0.0)
    Dc = spd_field(cfg.ncell, 7)
    Dc[::4] = 0.0
    z = inputs.uniform(cfg.ndofs, 8)
    y = run(cfg, z, (1, 0, 0), Dcell=Dc)
    yref, _ = o1.apply(*cfg.args(), z, periodic=(1, 0, 0), Dcell=Dc)
    assert np.all(np.isfinite(y))
    assert rel(y, yref) < TOL


@pytest.mark.parametrize("ncells", [(1, 1, 1), (1, 2, 3)])
def test_percell_single_cell_periodic(ncells):
    cfg = configs.small(3, ncells=ncells, hi=(0.5, 1.0, 0.75))
    Dc = spd_field(cfg.ncell, 3)
    z = inputs.uniform(cfg.ndofs, 5)
    y = run(cfg, z, (1, 1, 1), Dcell=Dc)
    yref, _ = o1.apply(*cfg.args(), z, periodic=(1, 1, 1), Dcell=Dc)
    assert rel(y, yref) < TOL


@pytest.mark.parametrize("k", [1, 3, 6])
def test_residual_consistency_discontinuous_D(k):
    """dg_residual(z*, F) ~ 0 for a continuous piecewise-linear u* whose normal flux is
    continuous across the jumps of a per-cell tensor (tests/test_oracle_next1.py)."""
    from oracle import rhs
    from paper_1711_10885_b200 import dg
    nc, lo, hi = (4, 2, 2), (0.0, 0.0, 0.0), (1.0, 0.5, 0.5)
    layers = spd_field(4, 31 + k)
    Dc = np.stack([layers[e % 4] for e in range(16)])
    field = rhs.KinkedField(lo[0], 0.25, layers[:, 0, 0], flux=1.3, u0=-0.4)
    args = (nc, lo, hi, k, (1, 0, 0, 0, 1, 0, 0, 0, 1), (0.7, -0.2, 0.5), 0.9, 3.0 * k * (k + 2) / 0.25)
    zs, F = rhs.consistency_data(*args, Dcell=Dc, field=field)
    op = dg.Operator(*args)
    op.set_diffusion(torch.from_numpy(Dc.reshape(-1)).cuda())
    zt, ft = torch.from_numpy(zs).cuda(), torch.from_numpy(F).cuda()
    r = torch.empty_like(zt)
    op.residual(zt, ft, r)
    torch.cuda.synchronize()
    op.close()
    assert np.abs(r.cpu().numpy()).max() < 1e-12 * np.abs(F).max()


def test_diagonal_field_matches_fast_kernel_and_revert():
    from paper_1711_10885_b200 import dg
    cfg = configs.small(7, ncells=(4, 4, 3), hi=(1.0, 1.0, 0.75))
    z = torch.from_numpy(inputs.uniform(cfg.ndofs, 12)).cuda()
    op = dg.from_config(cfg)
    y_fast = torch.empty_like(z)
    op.apply(z, y_fast)
    Dc = np.tile(np.asarray(cfg.D, float).reshape(1, 9), (cfg.ncell, 1))
    op.set_diffusion(torch.from_numpy(Dc.reshape(-1)).cuda())
    y_gen = torch.empty_like(z)
    op.apply(z, y_gen)
    op.set_diffusion(None)
    y_back = torch.empty_like(z)
    op.apply(z, y_back)
    torch.cuda.synchronize()
    op.close()
    a, b, c = (t.cpu().numpy() for t in (y_fast, y_gen, y_back))
    assert rel(b, a) < TOL
    assert np.array_equal(a, c)


def test_set_diffusion_rejects_bad_tensors():
    from paper_1711_10885_b200 import dg
    cfg = configs.small(2)
    op = dg.from_config(cfg)
    Dc = spd_field(cfg.ncell, 1)
    Dc[3, 0, 1] += 0.1                       # not symmetric
    with pytest.raises(dg.DGError) as ei:
        op.set_diffusion(torch.from_numpy(Dc.reshape(-1)).cuda())
    assert ei.value.code == dg.DG_EINVAL
    Dc = spd_field(cfg.ncell, 1)
    Dc[0, 2, 2] = -1.0                       # negative diagonal
    with pytest.raises(dg.DGError):
        op.set_diffusion(torch.from_numpy(Dc.reshape(-1)).cuda())
    Dc = spd_field(cfg.ncell, 1)
    Dc[5] = [[1.0, 2.0, 0.0], [2.0, 1.0, 0.0], [0.0, 0.0, 1.0]]   # indefinite, positive diagonal
    with pytest.raises(dg.DGError) as ei:
        op.set_diffusion(torch.from_numpy(Dc.reshape(-1)).cuda())
    assert ei.value.code == dg.DG_EINVAL
    op.close()


def test_rejected_set_diffusion_keeps_previous_field():
    """A rejected field leaves the operator as it was (validated before it is committed)."""
    from paper_1711_10885_b200 import dg
    cfg = configs.small(3, ncells=(3, 3, 2))
    op = dg.from_config(cfg)
    z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
    op.fill_uniform_local(z, 5)
    y0, y1 = torch.empty_like(z), torch.empty_like(z)
    good = spd_field(cfg.ncell, 2)
    op.set_diffusion(torch.from_numpy(good.reshape(-1)).cuda())
    op.apply(z, y0)
    bad = spd_field(cfg.ncell, 9)
    bad[4, 0, 1] += 0.5                      # not symmetric: rejected
    with pytest.raises(dg.DGError):
        op.set_diffusion(torch.from_numpy(bad.reshape(-1)).cuda())
    op.apply(z, y1)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    yo, _ = o1.apply(*cfg.args(), z.cpu().numpy(), Dcell=good)
    assert rel(y1.cpu().numpy(), yo) < TOL
    op.close()


def test_misaligned_vectors_rejected():
    """16-byte alignment is checked at the boundary (include/dg.h), not left to fault."""
    from paper_1711_10885_b200 import dg
    cfg = configs.small(7, ncells=(2, 2, 2))
    op = dg.from_config(cfg)
    buf = torch.zeros(op.ndofs + 2, dtype=torch.float64, device="cuda")
    y = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        op.apply(buf[1:1 + op.ndofs], y)
    L = dg.lib()
    assert L.dg_apply(op._h, dg._ptr(buf[1:]), dg._ptr(y), None) == dg.DG_EINVAL
    assert L.dg_apply(op._h, dg._ptr(buf[2:]), dg._ptr(y), None) == dg.DG_OK
    torch.cuda.synchronize()
    op.close()


@pytest.mark.slow
def test_problem_a_k7_sampled_vs_o1():
    """Problem-A-shaped run at k=7 (periodic, per-cell SPD tensors) on 64x32x32 cells, sampled."""
    from paper_1711_10885_b200 import dg
    cfg = configs.small(7, ncells=(64, 32, 32), hi=(2.0, 1.0, 1.0), b=(1.0, 0.5, 0.25), c=1.0)
    Dc = spd_field(cfg.ncell, 77)
    op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma,
                     bc=dg.bc_from_periodic((1, 1, 1)))
    op.set_diffusion(torch.from_numpy(Dc.reshape(-1)).cuda())
    z = torch.empty(cfg.ndofs, dtype=torch.float64, device="cuda")
    op.fill_uniform_local(z, 3)
    y = torch.empty_like(z)
    op.apply(z, y)
    torch.cuda.synchronize()
    op.close()
    zn, yn = z.cpu().numpy(), y.cpu().numpy()
    rng = np.random.default_rng(0)
    nx, ny, nz = cfg.ncells
    cells = np.unique(np.r_[[0, nx - 1, nx * ny - 1, cfg.ncell - 1], rng.integers(0, cfg.ncell, 200)]).astype(np.int64)
    ys, _ = o1.apply(*cfg.args(), zn, cells=cells, periodic=(1, 1, 1), Dcell=Dc)
    assert np.abs(yn.reshape(-1, cfg.n3)[cells] - ys).max() <= TOL * np.abs(yn).max()


def test_device_tensor_field_matches_host_recipe():
    from paper_1711_10885_b200 import dg
    cfg = configs.small(2, ncells=(5, 4, 3))
    # rank 1 of a 1x2x1 split (halo driven by the caller: no NCCL): global != local cell index
    op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma, rank=1, nranks=2,
                     parts=(1, 2, 1))
    u6 = torch.empty(op.ndofs // op.n3 * 6, dtype=torch.float64, device="cuda")
    op.fill_uniform_cells(u6, 6, 6)
    D_dev = inputs.tensor_field_from_uniforms(u6.view(-1, 6)).cpu().numpy()
    lo, cnt = op.cell_lo, op.cell_cnt
    gz, gy, gx = np.meshgrid(np.arange(lo[2], lo[2] + cnt[2]), np.arange(lo[1], lo[1] + cnt[1]),
                             np.arange(lo[0], lo[0] + cnt[0]), indexing="ij")
    own = (gx + cfg.ncells[0] * (gy + cfg.ncells[1] * gz)).reshape(-1)
    assert np.array_equal(D_dev, inputs.tensor_field_cells(own, 6))
    op.close()


# ------------------------------------------------------------------ NEXT-2: fused SSP-RK stages
@pytest.mark.parametrize("general,periodic,k", [(False, (0, 0, 0), 2), (False, (1, 1, 1), 7), (True, (1, 0, 1), 3),
                                                (True, (0, 0, 0), 7)])
def test_ssp_stages_vs_oracle(general, periodic, k):
    """Euler and Heun stages (out = a w + b (z + dt M^-1 (f - A z))) fused into
    the kernel's store, against O-1 + the same arithmetic written out in oracle/o1.ssp_stage."""
    from paper_1711_10885_b200 import dg
    cfg = configs.small(k, ncells=(4, 3, 2), hi=(1.0, 0.75, 0.5), b=(-0.8, 0.4, 0.3), c=0.6)
    Dc = spd_field(cfg.ncell, 9) if general else None
    op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma,
                     bc=dg.bc_from_periodic(periodic))
    if general:
        op.set_diffusion(torch.from_numpy(Dc.reshape(-1)).cuda())
    zn, fn = inputs.uniform(cfg.ndofs, 1), inputs.uniform(cfg.ndofs, 2)
    z, f = torch.from_numpy(zn).cuda(), torch.from_numpy(fn).cuda()
    dt = 2e-4
    e1 = torch.full_like(z, float("nan"))
    op.ssp_stage(z, e1, dt, f=f)
    h2 = torch.full_like(z, float("nan"))
    op.ssp_stage(e1, h2, dt, f=f, w=z, a=0.5, b=0.5)
    h3 = torch.full_like(z, float("nan"))
    op.heun_step(z, dt, torch.empty_like(z), h3, f=f)
    torch.cuda.synchronize()
    op.close()
    kw = {"periodic": periodic, "Dcell": Dc}
    e1r = o1.ssp_stage(*cfg.args(), zn, dt, f=fn, **kw)
    h2r = o1.ssp_stage(*cfg.args(), e1.cpu().numpy(), dt, f=fn, w=zn, a=0.5, bcoef=0.5, **kw)
    assert rel(e1.cpu().numpy(), e1r) < TOL
    assert rel(h2.cpu().numpy(), h2r) < TOL
    assert np.array_equal(h2.cpu().numpy(), h3.cpu().numpy())


def test_ssp_gpu_conserves_mass_periodic():
    """Periodic, c = 0, f = 0: 100 Heun steps keep sum_e z_(e,0) to rounding."""
    from paper_1711_10885_b200 import dg
    cfg = configs.small(5, ncells=(4, 4, 4), hi=(1.0, 1.0, 1.0), b=(1.0, -0.5, 0.25), c=0.0)
    op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma,
                     bc=dg.bc_from_periodic((1, 1, 1)))
    op.set_diffusion(torch.from_numpy(spd_field(cfg.ncell, 4).reshape(-1) * 1e-3).cuda())
    u = torch.from_numpy(inputs.uniform(cfg.ndofs, 3)).cuda()
    m0 = float(u.view(cfg.ncell, -1)[:, 0].sum())
    tmp, nxt = torch.empty_like(u), torch.empty_like(u)
    for _ in range(100):
        op.heun_step(u, 1e-4, tmp, nxt)
        u, nxt = nxt, u
    torch.cuda.synchronize()
    op.close()
    m1 = float(u.view(cfg.ncell, -1)[:, 0].sum())
    assert np.isfinite(m1) and abs(m1 - m0) < 1e-12 * float(u.abs().sum())


def test_general_kernel_symmetry_and_energy():
    """Invariants on the general kernel: SIPG symmetry for b = 0 with per-cell tensors on a periodic
    box (w^T A z = z^T A w), and for D = 0, c = 0 the pure-upwind energy z^T A z (positive: the
    upwind flux only dissipates) equal to O-1's."""
    from paper_1711_10885_b200 import dg
    cfg = configs.small(4, ncells=(4, 3, 3), hi=(1.0, 0.75, 0.75), b=(0, 0, 0), c=0.5)
    Dc = spd_field(cfg.ncell, 12)
    z = inputs.uniform(cfg.ndofs, 1)
    w = inputs.uniform(cfg.ndofs, 2)
    yz = run(cfg, z, (1, 1, 1), Dcell=Dc)
    yw = run(cfg, w, (1, 1, 1), Dcell=Dc)
    assert abs(w @ yz - z @ yw) < 1e-13 * abs(w @ yz)
    cfg2 = configs.small(3, ncells=(4, 3, 2), hi=(1.0, 0.75, 0.5), D=(0,) * 9, b=(1.0, -0.5, 0.25), c=0.0)
    op = dg.Operator(cfg2.ncells, cfg2.lo, cfg2.hi, cfg2.k, (0.1, 0.1, 0, 0.1, 0.1, 0, 0, 0, 0), cfg2.b, 0.0,
                     cfg2.sigma, bc=dg.bc_from_periodic((1, 1, 1)))   # off-diagonal (PSD) D: the general kernel
    op.set_diffusion(torch.zeros(cfg2.ncell * 9, dtype=torch.float64, device="cuda"))
    zz = inputs.uniform(cfg2.ndofs, 3)
    zt = torch.from_numpy(zz).cuda()
    y = torch.empty_like(zt)
    op.apply(zt, y)
    torch.cuda.synchronize()
    op.close()
    yref, _ = o1.apply(*cfg2.args(), zz, periodic=(1, 1, 1))
    E = zz @ yref
    assert E > 0 and abs(zz @ y.cpu().numpy() - E) < 1e-12 * E
