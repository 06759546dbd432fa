"""The direct (fused) halo between PROCESSES: dg_p2p_export / dg_p2p_import (CUDA IPC mappings of
the neighbours' receive buffers, IPC events, shared-memory counters). Two and four rank processes
share this box's one GPU (no NCCL: ncclCommInitRank refuses two ranks on one device; the ranks'
setup takes no ncclUniqueId, and no kernel waits on another -- every cross-rank dependency is a
stream wait on an IPC event recorded before it, B200_PROFILING.md). The trace pack kernel of each
rank stores straight into the neighbour's buffer; the gathered y of three consecutive applies
must equal the single-rank y bit for bit and O-1 at 1e-12."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, k, ncells, parts, periodic, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_10885_b200 import configs, dg
        torch.cuda.set_device(0)
        cfg = configs.small(k, ncells=ncells, hi=(1.5, 1.0, 0.75), b=(1.0, -0.5, 0.25), c=0.3)
        op = dg.Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma, device=0, rank=rank,
                         nranks=world, parts=parts, nccl_id=None, bc=dg.bc_from_periodic(periodic))
        dg.p2p_attach(op)
        transport = op.comm_info()
        z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
        y = torch.empty_like(z)
        outs = []
        for sd in range(3):
            op.fill_uniform_local(z, cfg.seed + sd)
            y.fill_(float("nan"))
            op.apply(z, y)
            outs.append(y.cpu().numpy().copy())
        op.sync()
        gathered = [None] * world
        dist.all_gather_object(gathered, (op.cell_lo, op.cell_cnt, outs, transport))
        op.close()
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k,ncells,parts,periodic", [
    (3, (4, 4, 2), (2, 1, 1), (0, 0, 0)),
    (7, (4, 2, 2), (2, 1, 1), (1, 0, 0)),     # two ranks along a periodic direction: both faces to one peer
    (2, (4, 4, 2), (2, 2, 1), (1, 1, 0)),
])
def test_ipc_direct_halo_equals_single_and_oracle(k, ncells, parts, periodic):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import o1
    from paper_1711_10885_b200 import configs, dg, inputs
    world = parts[0] * parts[1] * parts[2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, k, ncells, parts, periodic, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = configs.small(k, ncells=ncells, hi=(1.5, 1.0, 0.75), b=(1.0, -0.5, 0.25), c=0.3)
    G, n3 = cfg.ncells, cfg.n3
    op = dg.from_config(cfg, bc=dg.bc_from_periodic(periodic))
    z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(z)
    for sd in range(3):
        yg = np.full(cfg.ndofs, np.nan)
        for lo, cnt, outs, transport in gathered:
            assert transport == ("p2p-ipc", world)
            gz, gy, gx = np.meshgrid(np.arange(lo[2], lo[2] + cnt[2]), np.arange(lo[1], lo[1] + cnt[1]),
                                     np.arange(lo[0], lo[0] + cnt[0]), indexing="ij")
            yg.reshape(-1, n3)[(gx + G[0] * (gy + G[1] * gz)).reshape(-1)] = outs[sd].reshape(-1, n3)
        op.fill_uniform_local(z, cfg.seed + sd)
        op.apply(z, y)
        torch.cuda.synchronize()
        assert np.array_equal(yg, y.cpu().numpy()), sd
        yo, _ = o1.apply(*cfg.args(), inputs.uniform(cfg.ndofs, cfg.seed + sd), periodic=periodic)
        assert np.abs(yg - yo).max() <= 1e-12 * np.abs(yo).max()
    op.close()
