"""Randomised parity sweep on the GPU: seeded random combinations of degree, mesh shape (1..5
cells per direction, anisotropic boxes), boundary kinds (periodic / Dirichlet per direction),
coefficients (diagonal, full SPD or per-cell tensors; convection of either sign; reaction),
term masks and, for k <= 8, the variable-velocity kernel with or without over-integration —
each against the oracle O-1 element by element at the north_star tolerance 1e-12 (reading
C-14). Every kernel the operator can select (register-resident, pencil, general, velocity) is
reached by some case; the case list is fixed by the seeds, so a failure is reproducible."""
import numpy as np
import pytest

from oracle import o1
from paper_1711_10885_b200 import configs, inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def spd(rng):
    M = rng.normal(size=(3, 3))
    return M @ M.T + 0.3 * np.eye(3)


def case(seed):
    rng = np.random.default_rng(1000 + seed)
    k = int(rng.integers(1, 11))
    while True:
        nc = tuple(int(v) for v in rng.integers(1, 6, size=3))
        if nc[0] * nc[1] * nc[2] <= (40 if k <= 6 else 18):
            break
    lo = tuple(float(v) for v in rng.uniform(-1, 1, size=3))
    hi = tuple(lo[q] + float(rng.uniform(0.3, 1.5)) for q in range(3))
    periodic = tuple(int(v) for v in rng.integers(0, 2, size=3))
    kindD = int(rng.choice([0, 0, 0, 1, 2]))  # 0 diagonal, 1 full constant SPD, 2 per-cell tensors
    D = np.diag(rng.uniform(0.2, 2.0, size=3)) if kindD == 0 else spd(rng)
    b = tuple(float(v) for v in rng.uniform(-1.5, 1.5, size=3))
    c = float(rng.uniform(0, 1))
    velocity = k <= 8 and kindD == 0 and rng.uniform() < 0.3
    m = (k + 3 if rng.uniform() < 0.5 else k + 1) if velocity else 0
    if velocity:
        periodic = (0, 0, 0)                 # the linear test field is not box-periodic
    mask = int(rng.choice([7, 7, 1, 2, 4]))
    return k, nc, lo, hi, periodic, kindD, D, b, c, velocity, m, mask, rng


@pytest.mark.parametrize("seed", list(range(200)))
def test_random_case_vs_o1(seed):
    from paper_1711_10885_b200 import dg
    k, nc, lo, hi, periodic, kindD, D, b, c, velocity, m, mask, rng = case(seed)
    h = [(hi[q] - lo[q]) / nc[q] for q in range(3)]
    sigma = configs.sigma_for(k, min(h))
    ncell = nc[0] * nc[1] * nc[2]
    op = dg.Operator(nc, lo, hi, k, D.ravel(), b, c, sigma, bc=dg.bc_from_periodic(periodic))
    Dcell = None
    if kindD == 2:
        Dcell = np.stack([spd(rng) for _ in range(ncell)])
        op.set_diffusion(torch.from_numpy(np.ascontiguousarray(Dcell).reshape(-1)).cuda())
    if velocity:
        op.set_velocity(2)
        op.set_quadrature(m)
    n3 = (k + 1) ** 3
    z = inputs.uniform(ncell * n3, 77 + seed)
    zt = torch.from_numpy(z).cuda()
    y = torch.full_like(zt, float("nan"))
    op.apply(zt, y, terms=mask)
    torch.cuda.synchronize()
    op.close()
    yref, _ = o1.apply(nc, lo, hi, k, D.ravel(), b, c, sigma, z, mask=mask, periodic=periodic, Dcell=Dcell,
                       m=m, bkind=2 if velocity else 0)
    scale = np.abs(yref).max()
    yg = y.cpu().numpy()
    if scale == 0.0:
        assert np.abs(yg).max() == 0.0
    else:
        assert np.abs(yg - yref).max() / scale < TOL, (k, nc, periodic, kindD, velocity, m, mask)


@pytest.mark.parametrize("seed", list(range(40)))
def test_random_epilogues_vs_o1(seed):
    """The fused store epilogues on random cases: dg_residual r = f - A z and the SSP-RK stage
    out = a w + b (z + dt / Delta_T (f - A z)), from O-1's A z."""
    from paper_1711_10885_b200 import dg
    k, nc, lo, hi, periodic, kindD, D, b, c, velocity, m, mask, rng = case(5000 + seed)
    h = [(hi[q] - lo[q]) / nc[q] for q in range(3)]
    sigma = configs.sigma_for(k, min(h))
    ncell = nc[0] * nc[1] * nc[2]
    op = dg.Operator(nc, lo, hi, k, D.ravel(), b, c, sigma, bc=dg.bc_from_periodic(periodic))
    Dcell = None
    if kindD == 2:
        Dcell = np.stack([spd(rng) for _ in range(ncell)])
        op.set_diffusion(torch.from_numpy(np.ascontiguousarray(Dcell).reshape(-1)).cuda())
    if velocity:
        op.set_velocity(2)
        op.set_quadrature(m)
    n = ncell * (k + 1) ** 3
    z, f, w = inputs.uniform(n, 1 + seed), inputs.uniform(n, 2 + seed), inputs.uniform(n, 3 + seed)
    zt, ft, wt = (torch.from_numpy(v).cuda() for v in (z, f, w))
    r = torch.full_like(zt, float("nan"))
    op.residual(zt, ft, r)
    dt, a_, b_ = 1e-3 * float(rng.uniform(0.5, 2)), float(rng.uniform(0, 1)), float(rng.uniform(0.5, 1))
    out = torch.full_like(zt, float("nan"))
    op.ssp_stage(zt, out, dt, f=ft, w=wt, a=a_, b=b_)
    torch.cuda.synchronize()
    op.close()
    Az, _ = o1.apply(nc, lo, hi, k, D.ravel(), b, c, sigma, z, periodic=periodic, Dcell=Dcell, m=m,
                     bkind=2 if velocity else 0)
    rref = f - Az
    assert np.abs(r.cpu().numpy() - rref).max() <= TOL * np.abs(Az).max() + 1e-15
    dT = h[0] * h[1] * h[2]
    oref = a_ * w + b_ * (z + dt / dT * rref)
    assert np.abs(out.cpu().numpy() - oref).max() <= TOL * b_ * dt / dT * np.abs(Az).max() + 1e-14
