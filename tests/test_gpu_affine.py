"""NEXT-3 affine geometry on the GPU: dg_set_affine (the kernels integrate on the axis-aligned
reference mesh with the transformed coefficients and per-direction penalty) against O-2, which
evaluates every integral on the PHYSICAL mesh x = lo + J (xhat - lo); at 1e-12 (reading C-14)."""
import numpy as np
import pytest

from oracle import o2_assembled as o2, rhs
from paper_1711_10885_b200 import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-12

MESH = ((3, 2, 2), (0.0, 0.0, 0.0), (1.5, 1.0, 0.5))
SHEAR = np.array([[1.0, 0.3, 0.0], [0.0, 0.9, -0.2], [0.1, 0.0, 1.2]])
SCALE = np.diag([1.3, 0.8, 1.1])        # stays diagonal: the fast kernel
th = 0.5
ROT = np.array([[np.cos(th), -np.sin(th), 0.0], [np.sin(th), np.cos(th), 0.0], [0.0, 0.0, 1.0]])
DFULL = np.array([[1.0, 0.2, 0.0], [0.2, 2.0, 0.1], [0.0, 0.1, 0.5]])


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def op_for(k, D, b, c, sigma, J, periodic=(0, 0, 0)):
    from paper_1711_10885_b200 import dg
    nc, lo, hi = MESH
    op = dg.Operator(nc, lo, hi, k, D, b, c, sigma, bc=dg.bc_from_periodic(periodic))
    op.set_affine(J)
    return op


@pytest.mark.parametrize("J", [SHEAR, SCALE, ROT], ids=["shear", "scale", "rotation"])
@pytest.mark.parametrize("k,D", [(1, np.diag([1.0, 2.0, 0.5])), (2, DFULL), (3, np.diag([1.0, 2.0, 0.5]))])
@pytest.mark.parametrize("periodic", [(0, 0, 0), (1, 0, 1)])
def test_affine_vs_o2(J, k, D, periodic):
    nc, lo, hi = MESH
    b, c, sigma = (0.7, -0.4, 0.3), 0.6, 3.0 * k * (k + 2) / 0.25
    z = inputs.uniform(12 * (k + 1) ** 3, 31 + k)
    op = op_for(k, D, b, c, sigma, J, periodic)
    zt = torch.from_numpy(z).cuda()
    for mask in (7, 1, 2, 4):
        y = torch.full_like(zt, float("nan"))
        op.apply(zt, y, terms=mask)
        torch.cuda.synchronize()
        A = o2.assemble(nc, lo, hi, k, D, b, c, sigma, mask=mask, periodic=periodic, J=J)
        yref = A @ z
        if np.abs(yref).max() == 0:
            assert np.abs(y.cpu().numpy()).max() == 0
        else:
            assert rel(y.cpu().numpy(), yref) < TOL, mask
    op.close()


@pytest.mark.parametrize("k", [1, 2, 3])
def test_affine_residual_consistency(k):
    nc, lo, hi = MESH
    sigma = 3.0 * k * (k + 2) / 0.25
    args = (nc, lo, hi, k, DFULL, (0.7, -0.4, 0.3), 0.6, sigma)
    zs, F = rhs.consistency_data_affine(*args, SHEAR, seed=k)
    op = op_for(k, DFULL, (0.7, -0.4, 0.3), 0.6, sigma, SHEAR)
    zt, ft = torch.from_numpy(zs).cuda(), torch.from_numpy(F).cuda()
    r = torch.empty_like(zt)
    op.residual(zt, ft, r)
    torch.cuda.synchronize()
    op.close()
    assert np.abs(r.cpu().numpy()).max() < 1e-12 * np.abs(F).max()


def test_affine_percell_tensors_and_reset():
    """Per-cell physical tensors are mapped per cell; J = I afterwards restores nothing else
    (the per-cell field must be set after the map, so a new context is used for the check)."""
    nc, lo, hi = MESH
    k, b, c, sigma = 2, (0.7, -0.4, 0.3), 0.6, 60.0
    rng = np.random.default_rng(4)
    M = rng.normal(size=(12, 3, 3))
    Dc = np.einsum("eij,ekj->eik", M, M) + 0.5 * np.eye(3)
    z = inputs.uniform(12 * 27, 5)
    op = op_for(k, np.eye(3), b, c, sigma, SHEAR, (0, 1, 0))
    op.set_diffusion(torch.from_numpy(Dc.reshape(-1)).cuda())
    zt = torch.from_numpy(z).cuda()
    y = torch.empty_like(zt)
    op.apply(zt, y)
    torch.cuda.synchronize()
    A = o2.assemble(nc, lo, hi, k, np.eye(3), b, c, sigma, periodic=(0, 1, 0), Dcell=Dc, J=SHEAR)
    assert rel(y.cpu().numpy(), A @ z) < TOL
    from paper_1711_10885_b200 import dg
    with pytest.raises(dg.DGError):
        op.set_affine(np.eye(3))          # the map must precede per-cell tensors
    op.close()
    # identity map on a fresh context = the axis-aligned operator, bit for bit
    op1, op2 = op_for(k, DFULL, b, c, sigma, np.eye(3)), op_for(k, DFULL, b, c, sigma, SHEAR)
    op2.set_affine(np.eye(3))
    y1, y2 = torch.empty_like(zt), torch.empty_like(zt)
    op1.apply(zt, y1)
    op2.apply(zt, y2)
    torch.cuda.synchronize()
    assert np.array_equal(y1.cpu().numpy(), y2.cpu().numpy())
    op1.close()
    op2.close()


def test_affine_ssp_mass_matrix():
    """The explicit stage uses M = |J| Delta_T I on the affine mesh: pure reaction (D = 0, b = 0)
    gives z (1 - c dt) exactly as on the axis-aligned mesh."""
    k, c, dt = 3, 0.7, 0.2
    op = op_for(k, np.zeros(9), (0, 0, 0), c, 10.0, SHEAR)
    z = torch.from_numpy(inputs.uniform(12 * 64, 3)).cuda()
    out = torch.empty_like(z)
    op.ssp_stage(z, out, dt)
    torch.cuda.synchronize()
    op.close()
    assert rel(out.cpu().numpy(), z.cpu().numpy() * (1 - c * dt)) < 1e-14


@pytest.mark.parametrize("seed", list(range(15)))
def test_random_affine_vs_o2(seed):
    """Seeded random orientation-preserving affine maps, meshes, boundary kinds and coefficients
    (k <= 3, O-2 assembled on the physical mesh)."""
    rng = np.random.default_rng(900 + seed)
    k = int(rng.integers(1, 4))
    nc = tuple(int(v) for v in rng.integers(1, 4, size=3))
    lo = (0.0, 0.0, 0.0)
    hi = tuple(float(v) for v in rng.uniform(0.5, 1.5, size=3))
    while True:
        J = np.eye(3) + 0.4 * rng.normal(size=(3, 3))
        if np.linalg.det(J) > 0.2:
            break
    M = rng.normal(size=(3, 3))
    D = M @ M.T + 0.3 * np.eye(3)
    b = tuple(float(v) for v in rng.uniform(-1, 1, size=3))
    c = float(rng.uniform(0, 1))
    periodic = tuple(int(v) for v in rng.integers(0, 2, size=3))
    sigma = 3.0 * k * (k + 2) / min((hi[q] - lo[q]) / nc[q] for q in range(3))
    from paper_1711_10885_b200 import dg
    op = dg.Operator(nc, lo, hi, k, D.ravel(), b, c, sigma, bc=dg.bc_from_periodic(periodic))
    op.set_affine(J.ravel())
    n = nc[0] * nc[1] * nc[2] * (k + 1) ** 3
    z = inputs.uniform(n, 40 + seed)
    zt = torch.from_numpy(z).cuda()
    y = torch.full_like(zt, float("nan"))
    op.apply(zt, y)
    torch.cuda.synchronize()
    op.close()
    A = o2.assemble(nc, lo, hi, k, D, b, c, sigma, periodic=periodic, J=J)
    assert rel(y.cpu().numpy(), A @ z) < TOL, (k, nc, periodic)
