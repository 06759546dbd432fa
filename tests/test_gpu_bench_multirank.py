"""The N-rank bench path end to end on this box's one GPU: `python bench.py --gpus N --share-gpu`
launches N rank processes through torch.distributed.run (as the driver does for its scaling run),
each rank sets up its block of the partitioned mesh, attaches the direct IPC face-trace halo, runs
the timed applies, and rank 0 prints the contract JSON line after the max over ranks. --share-gpu
puts all ranks on one device with gloo instead of NCCL (ncclCommInitRank refuses two ranks on one
GPU); the pack kernels store into the neighbours' receive buffers exactly as across GPUs, and the
line's partition-invariance check (single-rank operator on 3x3x3-cell sub-boxes around sampled
cells, one next to every partition face) must be bitwise. Timing is not asserted."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# (8, c5weak): the driver's default N = 8 line (2 x 2 x 2 blocks of 128 x 128 x 64 cells, every rank with
# neighbours across all three partition directions)
@pytest.mark.parametrize("n,workload", [(2, "c3weak"), (4, "c3weak"), (2, "c5strong"), (8, "c5weak")])
def test_bench_n_ranks_on_one_gpu(n, workload):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--share-gpu", "--workload", workload,
           "--steps", "3", "--warmup", "3", "--no-e2e"]
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["shared_gpu"] is True
    assert d["comm"]["transport"] == "p2p-ipc" and d["comm"]["nranks"] == n
    par = d["parity"]
    assert par["cells_per_rank"] > 0 and par["bitwise"] and par["max_abs_err_over_max_abs_y"] == 0.0
    assert d["halo_ablation"]["ms_per_apply"] > 0 and d["value"] > 0
    assert d["config"]["parts"][0] * d["config"]["parts"][1] * d["config"]["parts"][2] == n
    # the overlap evidence: per rank, the pack (comm stream) and the inner / shell kernels (dg_timeline)
    tl = d["overlap_timeline"]["ms_since_apply_start"]
    assert len(tl) == n
    for t in tl:
        assert 0.0 <= t["pack_begin"] <= t["pack_end"]
        assert 0.0 <= t["inner_begin"] <= t["inner_end"]
        assert t["pack_end"] <= t["shell_begin"] <= t["shell_end"]   # the shell after its traces arrived
