"""NEXT-4 on the GPU: the assembled operator (dg_assemble,
probing the fused sum-factorized kernel) against the oracle O-2's entry-by-entry matrix, and the
matrix-based application (dg_matrix_apply) against O-1, both at the north_star tolerance 1e-12
(max-norm relative, reading C-14). The dense matrix is rebuilt from the block-stencil layout of
include/dg.h (dg_matrix_size) by adding every slot's block at its neighbour's columns."""
import numpy as np
import pytest

from oracle import o1, o2_assembled as o2
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


def neighbour(S, slot, nc, periodic):
    c = [S % nc[0], (S // nc[0]) % nc[1], S // (nc[0] * nc[1])]
    if slot > 0:
        q, s = (slot - 1) // 2, (slot - 1) % 2
        c[q] += 1 if s else -1
        if c[q] < 0 or c[q] >= nc[q]:
            if not periodic[q]:
                return None
            c[q] %= nc[q]
    return c[0] + nc[0] * (c[1] + nc[1] * c[2])


def dense_from_blocks(A, nc, n3, periodic):
    ncell = nc[0] * nc[1] * nc[2]
    ld = n3 + (n3 & 1)
    Ab = A.reshape(ncell, 7, n3, ld)           # [S][slot][column j][row i (padded to even)]
    assert not Ab[..., n3:].any(), "the pad row must be zero"
    Ab = Ab[..., :n3]
    M = np.zeros((ncell * n3, ncell * n3))
    for S in range(ncell):
        seen = set()
        for slot in range(7):
            T = neighbour(S, slot, nc, periodic)
            if T is None or T in seen:
                assert not Ab[S, slot].any(), "slot %d of cell %d must be zero" % (slot, S)
                continue
            seen.add(T)
            M[S * n3:(S + 1) * n3, T * n3:(T + 1) * n3] += Ab[S, slot].T
    return M


def make_op(cfg, periodic, Dcell=None, velocity=None, m=0, J=None):
    from paper_1711_10885_b200 import dg
    op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma,
                     bc=dg.bc_from_periodic(periodic))
    if J is not None:
        op.set_affine(J)
    if Dcell is not None:
        op.set_diffusion(torch.from_numpy(np.ascontiguousarray(Dcell, dtype=np.float64).reshape(-1)).cuda())
    if velocity is not None:
        op.set_velocity(velocity)
    if m:
        op.set_quadrature(m)
    return op


def assembled(op):
    A = torch.full((op.matrix_size(),), float("nan"), dtype=torch.float64, device="cuda")
    op.assemble(A)
    torch.cuda.synchronize()
    return A


def spd_field(ncell, seed):
    rng = np.random.default_rng(seed)
    M = rng.normal(size=(ncell, 3, 3))
    return np.einsum("eij,ekj->eik", M, M) + 0.5 * np.eye(3)[None]


CASES = [  # (k, ncells, periodic)
    (1, (3, 2, 2), (0, 0, 0)),
    (2, (3, 2, 2), (0, 0, 0)),
    (2, (4, 2, 1), (1, 1, 1)),     # periodic tails (4 = 3 + 1), 2 and 1 cells along a direction
    (1, (5, 1, 2), (1, 0, 1)),     # tail of 2 cells; a Dirichlet direction with 1 cell
    (3, (3, 3, 1), (1, 0, 1)),
    (1, (1, 1, 1), (1, 1, 1)),     # the cell is its own neighbour in every slot
]


@pytest.mark.parametrize("k,nc,periodic", CASES)
def test_assembled_matrix_vs_o2(k, nc, periodic):
    cfg = configs.small(k, ncells=nc, lo=(0.1, -0.2, 0.0), hi=(1.0, 0.6, 0.5), b=(1.0, -0.5, 0.25), c=0.3)
    op = make_op(cfg, periodic)
    A = assembled(op).cpu().numpy()
    op.close()
    M = dense_from_blocks(A, nc, (k + 1) ** 3, periodic)
    Aref = o2.assemble(*cfg.args(), periodic=periodic)
    assert rel(M, Aref) < TOL


def test_assembled_problem_a_vs_o2():
    # per-cell tensors, live weights and harmonic penalty (the matrix-based columns of Table 1
    # are Problem A's)
    k, nc, periodic = 2, (3, 2, 2), (1, 1, 1)
    cfg = configs.small(k, ncells=nc, hi=(0.75, 0.5, 0.5), b=(0.0, 0.0, 0.0), c=0.0)
    Dc = spd_field(12, 5)
    op = make_op(cfg, periodic, Dcell=Dc)
    A = assembled(op).cpu().numpy()
    op.close()
    M = dense_from_blocks(A, nc, (k + 1) ** 3, periodic)
    Aref = o2.assemble(*cfg.args(), periodic=periodic, Dcell=Dc)
    assert rel(M, Aref) < TOL
    assert rel(M, M.T) < TOL       # b = 0: symmetric


def test_assembled_velocity_field_overintegrated_vs_o2():
    k, nc = 2, (3, 2, 2)
    cfg = configs.small(k, ncells=nc, hi=(1.0, 0.5, 0.5), b=(1.0, 1.0, 1.0), c=0.2)
    op = make_op(cfg, (0, 0, 0), velocity=2, m=k + 3)
    A = assembled(op).cpu().numpy()
    op.close()
    M = dense_from_blocks(A, nc, (k + 1) ** 3, (0, 0, 0))
    Aref = o2.assemble(*cfg.args(), m=k + 3, bfield=o2.linear_field)
    assert rel(M, Aref) < TOL


def test_assembled_affine_vs_o2():
    k, nc, periodic = 2, (3, 2, 2), (0, 1, 0)
    J = ((1.0, 0.3, 0.0), (0.0, 1.0, 0.2), (0.1, 0.0, 0.9))
    cfg = configs.small(k, ncells=nc, hi=(0.75, 0.5, 0.5), D=(1.0, 0.2, 0.0, 0.2, 2.0, 0.1, 0.0, 0.1, 0.5),
                        b=(0.7, -0.4, 0.3), c=0.6)
    op = make_op(cfg, periodic, J=J)
    A = assembled(op).cpu().numpy()
    op.close()
    M = dense_from_blocks(A, nc, (k + 1) ** 3, periodic)
    Aref = o2.assemble(*cfg.args(), periodic=periodic, J=J)
    assert rel(M, Aref) < TOL


@pytest.mark.parametrize("periodic", [(0, 0, 0), (1, 0, 1)])
def test_assembled_multilinear_vs_o2g(periodic):
    """The assembled operator of a multilinear mesh (NEXT-3, q = 3p + 4) is the geometry oracle's
    matrix entry by entry (probing runs the geometry kernel)."""
    from oracle import o2_geometry as o2g
    from paper_1711_10885_b200 import dg, inputs
    k, nc, lo, hi = 2, (3, 3, 2), (0.0, 0.0, 0.0), (1.5, 1.5, 1.0)
    m = -(-(3 * k + 5) // 2)
    D = (1.0, 0.2, 0.1, 0.2, 2.0, -0.3, 0.1, -0.3, 0.5)
    op = dg.Operator(nc, lo, hi, k, D, (1.0, -0.5, 0.25), 0.3, 40.0, bc=dg.bc_from_periodic(periodic))
    box = ((-1, -1, -1), (nc[0] + 2, nc[1] + 2, nc[2] + 2))
    op.set_geometry(inputs.vertex_grid(nc, lo, hi, 0.2, 3, periodic, box=box), m)
    A = assembled(op).cpu().numpy()
    op.close()
    M = dense_from_blocks(A, nc, (k + 1) ** 3, periodic)
    Aref = o2g.assemble(nc, inputs.vertex_grid(nc, lo, hi, 0.2, 3, periodic), k, D, (1.0, -0.5, 0.25), 0.3, 40.0,
                        m=m, periodic=periodic)
    assert rel(M, Aref) < TOL


@pytest.mark.parametrize("k", [1, 3, 5, 7, 10])
@pytest.mark.parametrize("periodic", [(0, 0, 0), (1, 1, 1)])
def test_matrix_apply_vs_o1(k, periodic):
    nc = (4, 3, 2) if k < 10 else (3, 2, 2)
    cfg = configs.small(k, ncells=nc, lo=(0.1, -0.2, 0.0), hi=(1.0, 0.6, 0.5), b=(1.0, -0.5, 0.25), c=0.3)
    op = make_op(cfg, periodic)
    A = assembled(op)
    z_np = inputs.uniform(cfg.ndofs, 90 + k)
    z = torch.from_numpy(z_np).cuda()
    y = torch.full_like(z, float("nan"))
    ymf = torch.full_like(z, float("nan"))
    op.matrix_apply(A, z, y)
    op.apply(z, ymf)
    torch.cuda.synchronize()
    op.close()
    yref, _ = o1.apply(*cfg.args(), z_np, periodic=periodic)
    assert rel(y.cpu().numpy(), yref) < TOL
    assert rel(y.cpu().numpy(), ymf.cpu().numpy()) < TOL


@pytest.mark.parametrize("k,nc,periodic", [(1, (72, 64, 60), (0, 0, 0)), (2, (48, 40, 40), (1, 1, 1))])
def test_matrix_apply_large_vs_o1_sampled(k, nc, periodic):
    # enough row blocks for the unsplit launch (one CTA per 256 rows, all 7 slots); the
    # small meshes above take the slot-split path with the fixed-order reduction
    cfg = configs.small(k, ncells=nc, hi=(1.0, 1.0, 1.0), b=(1.0, -0.5, 0.25), c=0.3)
    op = make_op(cfg, periodic)
    A = assembled(op)
    z_np = inputs.uniform(cfg.ndofs, 60 + k)
    z = torch.from_numpy(z_np).cuda()
    y = torch.full_like(z, float("nan"))
    op.matrix_apply(A, z, y)
    torch.cuda.synchronize()
    op.close()
    ncell = nc[0] * nc[1] * nc[2]
    rng = np.random.default_rng(k)
    cells = np.unique(np.concatenate([rng.integers(0, ncell, 400), [0, ncell - 1, nc[0] - 1]])).astype(np.int64)
    yref, _ = o1.apply(*cfg.args(), z_np, cells=cells, periodic=periodic)
    n3 = (k + 1) ** 3
    yg = y.cpu().numpy().reshape(ncell, n3)[cells]
    assert rel(yg, yref) < TOL


def test_matrix_apply_repeat_deterministic():
    cfg = configs.small(3, ncells=(5, 4, 3), b=(1.0, -0.5, 0.25), c=0.3)
    op = make_op(cfg, (0, 0, 0))
    A = assembled(op)
    z = torch.from_numpy(inputs.uniform(cfg.ndofs, 3)).cuda()
    y1, y2 = torch.empty_like(z), torch.empty_like(z)
    op.matrix_apply(A, z, y1)
    op.matrix_apply(A, z, y2)
    torch.cuda.synchronize()
    op.close()
    assert torch.equal(y1, y2)


def test_matrix_argument_errors():
    from paper_1711_10885_b200 import dg
    cfg = configs.small(1, ncells=(2, 2, 2))
    op = make_op(cfg, (0, 0, 0))
    A = torch.zeros(op.matrix_size(), dtype=torch.float64, device="cuda")
    z = torch.zeros(cfg.ndofs, dtype=torch.float64, device="cuda")
    assert op.matrix_size() == 8 * 7 * 8 ** 2
    op3 = make_op(configs.small(2, ncells=(2, 1, 1)), (0, 0, 0))
    assert op3.matrix_size() == 2 * 7 * 27 * 28       # odd n^3: leading dimension padded to even
    op3.close()
    L = dg.lib()
    assert L.dg_matrix_apply(op._h, dg._ptr(A), dg._ptr(z), dg._ptr(z), None) == dg.DG_EINVAL   # y == z
    assert L.dg_matrix_apply(op._h, None, dg._ptr(z), dg._ptr(A), None) == dg.DG_EINVAL
    assert L.dg_assemble(op._h, None, None) == dg.DG_EINVAL
    op.close()


@pytest.mark.parametrize("seed", list(range(20)))
def test_random_matrix_apply_vs_o1(seed):
    """Seeded random meshes, boundary kinds, tensors and degrees: the assembled matrix applied
    to a vector equals O-1's y = A z (and the matrix-free apply) at 1e-12."""
    rng = np.random.default_rng(700 + seed)
    k = int(rng.integers(1, 8))
    nc = tuple(int(v) for v in rng.integers(1, 5, size=3))
    if k >= 5:
        nc = tuple(min(v, 2) for v in nc)
    periodic = tuple(int(v) for v in rng.integers(0, 2, size=3))
    cfg = configs.small(k, ncells=nc, lo=(0.0, -0.5, 0.2), hi=(1.2, 0.4, 0.9), b=tuple(rng.uniform(-1, 1, size=3)),
                        c=float(rng.uniform(0, 1)))
    Dc = spd_field(nc[0] * nc[1] * nc[2], seed) if rng.uniform() < 0.5 else None
    op = make_op(cfg, periodic, Dcell=Dc)
    A = assembled(op)
    z_np = inputs.uniform(cfg.ndofs, 11 + seed)
    z = torch.from_numpy(z_np).cuda()
    y = torch.full_like(z, float("nan"))
    op.matrix_apply(A, z, y)
    torch.cuda.synchronize()
    op.close()
    yref, _ = o1.apply(*cfg.args(), z_np, periodic=periodic, Dcell=Dc)
    assert rel(y.cpu().numpy(), yref) < TOL, (k, nc, periodic, Dc is not None)
