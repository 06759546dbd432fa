"""Multi-rank host logic on CPU (no GPU): world_size 2 (and 4) over torch.distributed gloo.

What runs on the GPU box with NCCL (bench.py --gpus N, dg_apply with nranks > 1) has
host-side ingredients that can be exercised here:
  * the block partition (dg_partition in the C ABI, the same rule dg_setup uses), including
    periodic wrap ranks,
  * the exchange pattern: one send/recv pair per partition face, the face layer ordered by the
    two tangential local coordinates (t1 fastest) as in include/dg.h.
Each rank computes its own cells with the ORACLE (O-1, sampled mode) from its own z plus the
neighbour ranks' face layers. The oracle evaluates neighbour traces itself, so what travels
here is the layer's z blocks; the library ships the face traces of those blocks (2 n^2 per
cell, include/dg.h), whose layout is pinned on the GPU against the oracle's own tables
(tests/test_gpu_loopback.py::test_trace_pack_layout_vs_oracle_tables). The gathered result
must equal the single-process oracle bit for bit.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def tangential(q):
    return (1, 2) if q == 0 else ((0, 2) if q == 1 else (0, 1))


def pack_layer(zloc, nloc, n3, face):
    """The face layer's z blocks, layer cells t1 fastest (the order of include/dg.h)."""
    q, s = face >> 1, face & 1
    t1, t2 = tangential(q)
    Z = zloc.reshape(nloc[2], nloc[1], nloc[0], n3)      # [z][y][x][j]
    idx = [slice(None)] * 3
    idx[2 - q] = nloc[q] - 1 if s else 0
    layer = Z[tuple(idx)]                                  # remaining axes ordered (z, y, x) minus q
    # remaining axes in (slow, fast) order are (t2, t1) because t1 < t2 and x is fastest
    return np.ascontiguousarray(layer).reshape(-1)


def worker(rank, world, port, parts, ncells, k, out_q, periodic=(0, 0, 0), percell=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import o1
        from paper_1711_10885_b200 import configs, dg, inputs

        cfg = configs.small(k, ncells=ncells, hi=(1.5, 1.0, 0.75), b=(1.0, -0.5, 0.25), c=0.3)
        n3 = cfg.n3
        lo, cnt, nbr = dg.partition(cfg.ncells, parts, rank, periodic)
        G = cfg.ncells
        # own cells (global ids) in local cell-major order
        gz, gy, gx = np.meshgrid(np.arange(lo[2], lo[2] + cnt[2]), np.arange(lo[1], lo[1] + cnt[1]),
                                 np.arange(lo[0], lo[0] + cnt[0]), indexing="ij")
        own = (gx + G[0] * (gy + G[1] * gz)).reshape(-1).astype(np.int64)
        zloc = inputs.uniform_cells(own, n3, cfg.seed).reshape(-1)
        Dglob = None
        if percell:   # the global field is a pure function of the seed; each rank keeps its own cells
            rng = np.random.default_rng(k)
            M = rng.normal(size=(cfg.ncell, 3, 3))
            Dglob = (np.einsum("eij,ekj->eik", M, M) + 0.5 * np.eye(3)).reshape(cfg.ncell, 9)
            Dloc = np.ascontiguousarray(Dglob[own]).reshape(-1)
        # halo exchange: one send/recv pair per partition face (gloo stands in for NCCL); with
        # periodic wrap and two ranks along a direction both faces go to the same peer (tags
        # keep the pairs apart, as the send f / receive f^1 issue order does for NCCL)
        recv, drecv = {}, {}
        reqs = []
        for f in range(6):
            if nbr[f] < 0:
                continue
            buf = torch.from_numpy(pack_layer(zloc, cnt, n3, f))
            q = f >> 1
            t1, t2 = tangential(q)
            rbuf = torch.empty(cnt[t1] * cnt[t2] * n3, dtype=torch.float64)
            recv[f] = rbuf
            reqs.append(dist.isend(buf, nbr[f], tag=f))
            reqs.append(dist.irecv(rbuf, nbr[f], tag=f ^ 1))
            if percell:
                dbuf = torch.from_numpy(pack_layer(Dloc, cnt, 9, f))
                drecv[f] = torch.empty(cnt[t1] * cnt[t2] * 9, dtype=torch.float64)
                reqs.append(dist.isend(dbuf, nbr[f], tag=16 + f))
                reqs.append(dist.irecv(drecv[f], nbr[f], tag=16 + (f ^ 1)))
        for r in reqs:
            r.wait()
        # extended global-shaped z: own cells + ghost layers, zeros elsewhere
        zext = np.zeros(cfg.ndofs)
        zext.reshape(-1, n3)[own] = zloc.reshape(-1, n3)
        Dext = None
        if percell:
            Dext = np.zeros((cfg.ncell, 9))
            Dext[own] = Dloc.reshape(-1, 9)
        for f, rbuf in recv.items():
            q, s = f >> 1, f & 1
            t1, t2 = tangential(q)
            lay = rbuf.numpy().reshape(cnt[t2], cnt[t1], n3)
            dlay = drecv[f].numpy().reshape(cnt[t2], cnt[t1], 9) if percell else None
            for i2 in range(cnt[t2]):
                for i1 in range(cnt[t1]):
                    g = [0, 0, 0]
                    g[q] = (lo[q] + cnt[q]) % G[q] if s else (lo[q] - 1) % G[q]
                    g[t1] = lo[t1] + i1
                    g[t2] = lo[t2] + i2
                    e = g[0] + G[0] * (g[1] + G[1] * g[2])
                    zext[e * n3:(e + 1) * n3] = lay[i2, i1]
                    if percell:
                        Dext[e] = dlay[i2, i1]
        yloc, _ = o1.apply(*cfg.args(), zext, cells=own, nthreads=1, periodic=periodic, Dcell=Dext)
        # gather to rank 0 and compare with the single-process oracle
        gathered = [None] * world
        dist.all_gather_object(gathered, (own, yloc))
        if rank == 0:
            full = inputs.uniform(cfg.ndofs, cfg.seed)
            yref, _ = o1.apply(*cfg.args(), full, nthreads=1, periodic=periodic, Dcell=Dglob)
            got = np.zeros_like(yref)
            seen = np.zeros(cfg.ncell, dtype=int)
            for cells, yl in gathered:
                got.reshape(-1, n3)[cells] = yl
                seen[cells] += 1
            out_q.put((bool(np.all(seen == 1)), bool(np.array_equal(got, yref)), list(nbr)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("parts,ncells,k", [((2, 1, 1), (4, 3, 2), 2), ((1, 2, 1), (3, 4, 2), 1),
                                            ((1, 1, 2), (2, 3, 4), 3), ((2, 2, 1), (4, 4, 2), 1)])
def test_partitioned_oracle_equals_global(parts, ncells, k):
    run_world(parts, ncells, k)


@pytest.mark.parametrize("parts,ncells,k,periodic", [((2, 1, 1), (4, 3, 2), 2, (1, 0, 0)),
                                                     ((2, 2, 1), (4, 4, 2), 1, (1, 1, 1)),
                                                     ((1, 1, 2), (2, 3, 4), 2, (0, 1, 1))])
def test_partitioned_periodic_percell_oracle_equals_global(parts, ncells, k, periodic):
    """NEXT-1 host logic: periodic wrap ranks (dg_partition) and the per-cell tensor layers."""
    run_world(parts, ncells, k, periodic, True)


def run_world(parts, ncells, k, periodic=(0, 0, 0), percell=False):
    world = parts[0] * parts[1] * parts[2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, parts, ncells, k, q, periodic, percell))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    covered, equal, _ = res
    assert covered, "partition does not tile the mesh exactly once"
    assert equal, "partitioned result differs from the single-rank result"


def test_partition_rule_properties():
    from paper_1711_10885_b200 import dg
    for parts in ((2, 1, 1), (2, 2, 1), (2, 2, 2), (1, 4, 2)):
        world = parts[0] * parts[1] * parts[2]
        ncells = (8, 8, 4)
        boxes = {}
        for r in range(world):
            lo, cnt, nbr = dg.partition(ncells, parts, r)
            boxes[r] = (lo, cnt, nbr)
            for f in range(6):
                if nbr[f] >= 0:
                    # symmetric neighbour relation across opposite faces
                    assert dg.partition(ncells, parts, nbr[f])[2][f ^ 1] == r
            assert r == (lo[0] // cnt[0]) + parts[0] * ((lo[1] // cnt[1]) + parts[1] * (lo[2] // cnt[2]))
        vol = sum(np.prod(b[1]) for b in boxes.values())
        assert vol == np.prod(ncells)
    with pytest.raises(Exception):
        dg.partition((8, 8, 4), (3, 1, 1), 0)


def test_partition_periodic_wrap():
    from paper_1711_10885_b200 import dg
    # two ranks along a periodic x: each is the other's neighbour on both x faces
    assert dg.partition((8, 4, 4), (2, 1, 1), 0, (1, 0, 0))[2][:2] == (1, 1)
    # periodic but unsplit: the wrap is local (no neighbour rank)
    assert dg.partition((8, 4, 4), (1, 2, 1), 0, (1, 1, 0))[2][:2] == (-1, -1)
    assert dg.partition((8, 4, 4), (1, 2, 1), 0, (1, 1, 0))[2][2:4] == (1, 1)
    # four ranks in a periodic ring along z
    nb = [dg.partition((4, 4, 8), (1, 1, 4), r, (0, 0, 1))[2][4:] for r in range(4)]
    assert nb == [(3, 1), (0, 2), (1, 3), (2, 0)]
