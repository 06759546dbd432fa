"""bench.py's reference arm (the oracle O-1 on the host cores) as the driver launches it at N > 1:
rank 0 alone prints the contract line for the N-GPU workload, timing rank 0's block of the
partition as a standalone mesh (the global z would not fit a host at N = 8); the other ranks exit 0
without output. CPU only (no torch.cuda)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(rank, world, workload):
    env = dict(os.environ, PYTHONPATH=ROOT, RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", str(world),
           "--workload", workload, "--steps", "1", "--warmup", "1", "--ref-seconds", "2"]
    return subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)


def test_reference_arm_rank0_block_line():
    r = _run(0, 2, "c3weak")
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["unit"] == "DOF/s" and d["higher_is_better"] is True
    assert "256x64x64" in d["config"]["workload"]               # the 2-GPU workload is what the line names
    assert "(rank 0 block)" in d["cpu_baseline"]["sample"]      # ... timed on rank 0's 128x64x64 block
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_silent():
    r = _run(1, 2, "c3weak")
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]
