"""Single-GPU loopback of the multi-rank path (SURVEY.md 4 "loopback partition test").

(1) P contexts (ranks of a Px x Py x Pz block partition) live on one device; each packs the
face traces of its partition layers with the library (dg_halo_pack), the test copies every
send buffer into the neighbour's receive buffer (no kernel waits on another), and each rank
applies with DG_HALO_EXTERNAL.
(2) The whole partitioned dg_apply, exchange included: the ranks are THREADS of this process
joined by the in-process fabric (dg_fabric_id), each calling dg_apply / dg_residual /
dg_ssp_stage / dg_set_diffusion on its own stream -- the trace pack on the comm stream, the
exchange (NCCL's per-peer issue-order matching), the inner-box kernel, the shell kernel after
the receive event, and the write-after-read guard across consecutive applies.
The gathered y must equal the single-rank y BIT FOR BIT (every cell runs the same arithmetic
whether its neighbour is local or a ghost: partition invariance) and the
oracle O-1 within 1e-12."""
import threading

import numpy as np
import pytest

from oracle import o1
from paper_1711_10885_b200 import configs, inputs

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
                dc = cnt // (2 * (cfg.k + 1) ** 2) * 6     # face traces: 2 n^2 per layer cell
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
        yo, _ = o1.apply(*cfg.args(), inputs.uniform(cfg.ndofs, cfg.seed), mask=terms)
        assert np.abs(yp - yo).max() <= 1e-12 * np.abs(yo).max()


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


# ------------------------------------------------------------------ (2) threads + in-process fabric
def gather(cfg, ops, per_rank):
    n3 = cfg.n3
    yg = np.full(cfg.ndofs, np.nan)
    for op, y in zip(ops, per_rank):
        yg.reshape(-1, n3)[local_cells(cfg, op.cell_lo, op.cell_cnt)] = y.reshape(-1, n3)
    return yg


def run_fabric(cfg, parts, periodic=(0, 0, 0), Dcell=None, seeds=(0,), mode="apply", direct=False):
    """Every rank on its own thread and stream; per seed one collective call. Returns the
    gathered result per seed. direct: the fused halo (the pack stores into the neighbours' receive
    buffers, dg_fabric_id_direct) instead of send buffers + copies."""
    from paper_1711_10885_b200 import dg
    world = parts[0] * parts[1] * parts[2]
    fid = dg.fabric_id_direct() if direct else dg.fabric_id()
    ops = [dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma, rank=r, nranks=world,
                       parts=parts, nccl_id=fid, bc=dg.bc_from_periodic(periodic)) for r in range(world)]
    out = [None] * world
    errors = []
    for op in ops:
        assert op.comm_info() == ("fabric-direct" if direct else "fabric", world)

    def work(r):
        try:
            op = ops[r]
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                if Dcell is not None:
                    own = local_cells(cfg, op.cell_lo, op.cell_cnt)
                    op.set_diffusion(torch.from_numpy(np.ascontiguousarray(Dcell[own]).reshape(-1)).cuda(), stream=st)
                z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
                y = torch.empty_like(z)
                f = torch.empty_like(z)
                res = []
                for sd in seeds:            # consecutive collective calls reuse z, y and the halo buffers
                    op.fill_uniform_local(z, cfg.seed + sd, stream=st)
                    y.fill_(float("nan"))
                    if mode == "apply":
                        op.apply(z, y, stream=st)
                    elif mode == "residual":
                        op.fill_uniform_local(f, 99 + sd, stream=st)
                        op.residual(z, f, y, stream=st)
                    else:                   # Heun stage 2 form: out = 1/2 w + 1/2 (z + dt M^-1 (f - A z))
                        op.fill_uniform_local(f, 77 + sd, stream=st)
                        op.ssp_stage(z, y, 1e-3, f=f, w=f, a=0.5, b=0.5, stream=st)
                    res.append(y.clone())
                st.synchronize()
                out[r] = [t.cpu().numpy() for t in res]
                op.sync()
        except Exception as e:  # noqa: BLE001 -- reported below
            errors.append((r, repr(e)))

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "fabric ranks hung"
    assert not errors, errors
    res = [gather(cfg, ops, [out[r][i] for r in range(world)]) for i in range(len(seeds))]
    for op in ops:
        op.close()
    return res


def single_fn(cfg, periodic, Dcell, mode):
    from paper_1711_10885_b200 import dg
    op = dg.from_config(cfg, bc=dg.bc_from_periodic(periodic))
    if Dcell is not None:
        op.set_diffusion(torch.from_numpy(np.ascontiguousarray(Dcell).reshape(-1)).cuda())
    z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(z)
    f = torch.empty_like(z)

    def run(sd):
        op.fill_uniform_local(z, cfg.seed + sd)
        if mode == "apply":
            op.apply(z, y)
        elif mode == "residual":
            op.fill_uniform_local(f, 99 + sd)
            op.residual(z, f, y)
        else:
            op.fill_uniform_local(f, 77 + sd)
            op.ssp_stage(z, y, 1e-3, f=f, w=f, a=0.5, b=0.5)
        torch.cuda.synchronize()
        return y.cpu().numpy().copy()
    return op, run


@pytest.mark.parametrize("k,ncells,parts,periodic", [
    (2, (6, 4, 4), (2, 1, 1), (0, 0, 0)), (3, (4, 4, 4), (2, 2, 1), (0, 0, 0)), (7, (4, 4, 4), (2, 2, 2), (0, 0, 0)),
    (7, (4, 2, 2), (2, 1, 1), (1, 0, 0)),          # two ranks along a periodic direction: both faces, one peer
    (3, (4, 4, 4), (2, 2, 2), (1, 1, 1)), (1, (4, 6, 8), (1, 2, 4), (0, 1, 1)), (10, (2, 2, 4), (1, 1, 2), (0, 0, 1)),
    (5, (2, 2, 2), (2, 2, 2), (1, 1, 1)),          # one cell per rank: every cell is a shell cell
])
@pytest.mark.parametrize("direct", [False, True])
def test_fabric_apply_equals_single_and_oracle(k, ncells, parts, periodic, direct):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = configs.small(k, ncells=ncells, hi=(1.5, 1.0, 0.75), b=(1.0, -0.5, 0.25), c=0.3)
    seeds = (0, 1, 2)
    yps = run_fabric(cfg, parts, periodic, seeds=seeds, direct=direct)
    op, run = single_fn(cfg, periodic, None, "apply")
    for sd, yp in zip(seeds, yps):
        assert np.array_equal(yp, run(sd)), sd
        yo, _ = o1.apply(*cfg.args(), inputs.uniform(cfg.ndofs, cfg.seed + sd), periodic=periodic)
        assert np.abs(yp - yo).max() <= 1e-12 * np.abs(yo).max(), sd
    op.close()


@pytest.mark.parametrize("mode", ["residual", "ssp"])
@pytest.mark.parametrize("direct", [False, True])
def test_fabric_epilogues(mode, direct):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = configs.small(4, ncells=(4, 4, 2), hi=(1.5, 1.0, 0.75), b=(1.0, -0.5, 0.25), c=0.3)
    yps = run_fabric(cfg, (2, 2, 1), (1, 0, 0), seeds=(0, 1), mode=mode, direct=direct)
    op, run = single_fn(cfg, (1, 0, 0), None, mode)
    for sd, yp in zip((0, 1), yps):
        assert np.array_equal(yp, run(sd))
    op.close()


@pytest.mark.parametrize("k,parts,periodic", [(2, (2, 2, 1), (1, 1, 0)), (7, (2, 1, 1), (1, 1, 1)),
                                              (3, (2, 2, 2), (0, 0, 0))])
@pytest.mark.parametrize("direct", [False, True])
def test_fabric_percell_tensors(k, parts, periodic, direct):
    """dg_set_diffusion exchanges the partition layers of the tensor field through the fabric
    (NEXT-1), then applies exchange the traces (copied, or stored directly by the pack)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = configs.small(k, ncells=(4, 2, 2) if k == 7 else (4, 4, 4), hi=(1.5, 1.0, 0.75), b=(1.0, -0.5, 0.25),
                        c=0.3)
    rng = np.random.default_rng(k)
    M = rng.normal(size=(cfg.ncell, 3, 3))
    Dc = (np.einsum("eij,ekj->eik", M, M) + 0.5 * np.eye(3)).reshape(cfg.ncell, 9)
    yps = run_fabric(cfg, parts, periodic, Dcell=Dc, seeds=(0, 1), direct=direct)
    op, run = single_fn(cfg, periodic, Dc, "apply")
    for sd, yp in zip((0, 1), yps):
        assert np.array_equal(yp, run(sd))
        yo, _ = o1.apply(*cfg.args(), inputs.uniform(cfg.ndofs, cfg.seed + sd), periodic=periodic,
                         Dcell=Dc.reshape(-1, 3, 3))
        assert np.abs(yp - yo).max() <= 1e-12 * np.abs(yo).max()
    op.close()


@pytest.mark.parametrize("k,ncells,parts", [(1, (4, 3, 2), (2, 1, 1)), (4, (2, 4, 3), (1, 2, 1)),
                                            (7, (3, 2, 4), (1, 1, 2)), (10, (2, 2, 2), (2, 2, 2))])
def test_trace_pack_layout_vs_oracle_tables(k, ncells, parts):
    """The halo payload (include/dg.h): per partition face f = 2q + s and layer cell
    t1 + N_t1 t2, [u | d][a + n b] with u = sum_e theta_e(s) z(e; a, b) and d the same with
    theta'_e(s) (the normal-first face contraction), written out here with the
    ORACLE's tables (o1.tables: theta(0), theta(1), theta'(0), theta'(1))."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1711_10885_b200 import dg
    cfg = configs.small(k, ncells=ncells)
    n = k + 1
    _, _, _, _, th0, th1, dth0, dth1 = o1.tables(k)
    world = parts[0] * parts[1] * parts[2]
    for r in range(world):
        op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma, rank=r, nranks=world,
                         parts=parts)
        z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
        op.fill_uniform_local(z, 3)
        op.halo_pack(z)
        torch.cuda.synchronize()
        cnt = op.cell_cnt
        Z = z.cpu().numpy().reshape(cnt[2], cnt[1], cnt[0], n, n, n)     # [cz][cy][cx][jz][jy][jx]
        for f in range(6):
            nb, count = op.halo_info(f)
            if nb < 0:
                continue
            q, s = f >> 1, f & 1
            t1, t2 = (1, 2) if q == 0 else ((0, 2) if q == 1 else (0, 1))
            assert count == cnt[t1] * cnt[t2] * 2 * n * n
            got = as_tensor(op.halo_buffer_ptr(f, 0), count).cpu().numpy().reshape(cnt[t2], cnt[t1], 2, n, n)
            th, dth = (th1, dth1) if s else (th0, dth0)
            # move axes to [c_t2][c_t1][c_q][j_t2][j_t1][j_q]  (array axes: c 0..2 = z,y,x; j 3..5 = z,y,x)
            ax = lambda d: 2 - d  # noqa: E731
            W = np.transpose(Z, (ax(t2), ax(t1), ax(q), 3 + ax(t2), 3 + ax(t1), 3 + ax(q)))
            lay = W[:, :, cnt[q] - 1 if s else 0]                            # [c_t2][c_t1][b][a][e]
            want_u = np.einsum("xyabe,e->xyab", lay, th)
            want_d = np.einsum("xyabe,e->xyab", lay, dth)
            assert np.allclose(got[:, :, 0], want_u, rtol=0, atol=1e-13 * max(1, np.abs(want_u).max()))
            assert np.allclose(got[:, :, 1], want_d, rtol=0, atol=1e-13 * max(1, np.abs(want_d).max()))
        op.close()
