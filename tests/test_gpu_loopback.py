"""Single-GPU loopback of the multi-rank path (SURVEY.md 4 "loopback partition test").

P contexts (ranks of a Px x Py x Pz block partition) live on one device; each packs its
partition layers with the library (dg_halo_pack), the test copies every send buffer into
the neighbour's receive buffer (standing in for the NCCL exchange; no kernel waits on
another), and each rank applies with DG_HALO_EXTERNAL. The gathered y must equal the
single-rank y BIT FOR BIT: every cell runs the same arithmetic whether its neighbour is
local or a ghost (partition invariance)."""
import numpy as np
import pytest

from paper_1711_10885_b200 import configs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


class DevPtr:
    """A raw device pointer as a torch tensor view (__cuda_array_interface__)."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def as_tensor(ptr, count):
    return torch.as_tensor(DevPtr(ptr, count), device="cuda")


def local_cells(cfg, lo, cnt):
    G = cfg.ncells
    gz, gy, gx = np.meshgrid(np.arange(lo[2], lo[2] + cnt[2]), np.arange(lo[1], lo[1] + cnt[1]),
                             np.arange(lo[0], lo[0] + cnt[0]), indexing="ij")
    return (gx + G[0] * (gy + G[1] * gz)).reshape(-1)


def run_partitioned(cfg, parts, terms, periodic=(0, 0, 0), Dcell=None):
    from paper_1711_10885_b200 import dg
    world = parts[0] * parts[1] * parts[2]
    ops, zs, ys = [], [], []
    for r in range(world):
        op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma, rank=r, nranks=world,
                         parts=parts, bc=dg.bc_from_periodic(periodic))
        if Dcell is not None:
            own = local_cells(cfg, op.cell_lo, op.cell_cnt)
            op.set_diffusion(torch.from_numpy(np.ascontiguousarray(Dcell[own]).reshape(-1)).cuda(),
                             flags=dg.HALO_EXTERNAL)
        z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
        op.fill_uniform_local(z, cfg.seed)
        op.halo_pack(z)
        ops.append(op)
        zs.append(z)
    torch.cuda.synchronize()
    for r, op in enumerate(ops):
        for f in range(6):
            nb, cnt = op.halo_info(f)
            if nb < 0:
                continue
            src = as_tensor(ops[nb].halo_buffer_ptr(f ^ 1, 0), cnt)
            dst = as_tensor(op.halo_buffer_ptr(f, 1), cnt)
            dst.copy_(src)
            if Dcell is not None:    # the diffusion-field layers (which = 2 / 3)
                dc = cnt // cfg.n3 * 6
                as_tensor(op.halo_buffer_ptr(f, 3), dc).copy_(as_tensor(ops[nb].halo_buffer_ptr(f ^ 1, 2), dc))
    torch.cuda.synchronize()
    n3 = cfg.n3
    G = cfg.ncells
    yg = np.full(cfg.ndofs, np.nan)
    for r, op in enumerate(ops):
        y = torch.full_like(zs[r], float("nan"))
        op.apply(zs[r], y, terms=terms | dg.HALO_EXTERNAL)
        torch.cuda.synchronize()
        lo, cnt = op.cell_lo, op.cell_cnt
        gz, gy, gx = np.meshgrid(np.arange(lo[2], lo[2] + cnt[2]), np.arange(lo[1], lo[1] + cnt[1]),
                                 np.arange(lo[0], lo[0] + cnt[0]), indexing="ij")
        own = (gx + G[0] * (gy + G[1] * gz)).reshape(-1)
        yg.reshape(-1, n3)[own] = y.cpu().numpy().reshape(-1, n3)
        ys.append(y)
    for op in ops:
        op.close()
    return yg


def run_single(cfg, terms, periodic=(0, 0, 0), Dcell=None):
    from paper_1711_10885_b200 import dg
    op = dg.from_config(cfg, bc=dg.bc_from_periodic(periodic))
    if Dcell is not None:
        op.set_diffusion(torch.from_numpy(np.ascontiguousarray(Dcell).reshape(-1)).cuda())
    z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
    op.fill_uniform_local(z, cfg.seed)
    y = torch.empty_like(z)
    op.apply(z, y, terms=terms)
    torch.cuda.synchronize()
    op.close()
    return y.cpu().numpy()


@pytest.mark.parametrize("k,ncells,parts", [
    (2, (6, 4, 4), (2, 1, 1)), (2, (6, 4, 4), (2, 2, 1)), (3, (4, 4, 4), (2, 2, 2)),
    (7, (4, 4, 4), (2, 2, 2)), (7, (8, 4, 2), (2, 2, 1)), (1, (4, 6, 8), (1, 2, 4)), (10, (2, 2, 4), (1, 1, 2)),
])
def test_partitioned_equals_single_bitwise(k, ncells, parts):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = configs.small(k, ncells=ncells, hi=(1.5, 1.0, 0.75), b=(1.0, -0.5, 0.25), c=0.3)
    for terms in (7, 2):
        ys = run_single(cfg, terms)
        yp = run_partitioned(cfg, parts, terms)
        assert np.array_equal(yp, ys)


@pytest.mark.parametrize("k,ncells,parts,periodic", [
    (2, (6, 4, 4), (2, 1, 1), (1, 0, 0)), (3, (4, 4, 4), (2, 2, 2), (1, 1, 1)), (7, (4, 4, 2), (2, 2, 1), (1, 1, 1)),
    (7, (4, 4, 2), (2, 2, 1), (0, 0, 1)), (1, (4, 6, 8), (1, 2, 4), (0, 1, 1)),
])
@pytest.mark.parametrize("percell", [False, True])
def test_partitioned_periodic_percell_equals_single_bitwise(k, ncells, parts, periodic, percell):
    """Periodic wrap across ranks (two ranks along a direction: both faces talk to the same
    peer) and per-cell tensors whose partition layers travel with the halo (NEXT-1)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = configs.small(k, ncells=ncells, hi=(1.5, 1.0, 0.75), b=(1.0, -0.5, 0.25), c=0.3)
    Dc = None
    if percell:
        rng = np.random.default_rng(k)
        M = rng.normal(size=(cfg.ncell, 3, 3))
        Dc = (np.einsum("eij,ekj->eik", M, M) + 0.5 * np.eye(3)).reshape(cfg.ncell, 9)
    for terms in (7, 2):
        ys = run_single(cfg, terms, periodic, Dc)
        yp = run_partitioned(cfg, parts, terms, periodic, Dc)
        assert np.array_equal(yp, ys)


@pytest.mark.parametrize("seed", list(range(30)))
def test_random_partitions_equal_single_bitwise(seed):
    """Seeded random partitions (1-2 ranks per direction, 1-3 cells per rank and direction),
    periodic sides, per-cell tensors and degrees: the partitioned result equals the single-rank
    one bit for bit (partition invariance)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(500 + seed)
    while True:
        parts = tuple(int(v) for v in rng.integers(1, 3, size=3))
        if parts[0] * parts[1] * parts[2] >= 2:
            break
    ncells = tuple(parts[q] * int(rng.integers(1, 4)) for q in range(3))
    k = int(rng.integers(1, 11))
    if k >= 8:
        ncells = tuple(min(v, 2 * parts[q]) for q, v in enumerate(ncells))
    periodic = tuple(int(v) for v in rng.integers(0, 2, size=3))
    percell = bool(rng.integers(0, 2))
    cfg = configs.small(k, ncells=ncells, hi=(1.5, 1.0, 0.75), b=tuple(rng.uniform(-1, 1, size=3)), c=0.3)
    Dc = None
    if percell:
        M = rng.normal(size=(cfg.ncells[0] * cfg.ncells[1] * cfg.ncells[2], 3, 3))
        Dc = np.einsum("eij,ekj->eik", M, M) + 0.5 * np.eye(3)[None]
    terms = int(rng.choice([7, 7, 2]))
    ys = run_single(cfg, terms, periodic, Dc)
    yp = run_partitioned(cfg, parts, terms, periodic, Dc)
    assert np.array_equal(yp, ys), (k, ncells, parts, periodic, percell, terms)
