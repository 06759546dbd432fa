"""Degree sweep (BASELINE config C4) and the large single-GPU configs, through the C ABI.

    python tools/sweep.py [--reps 10] [--out gpurun_out/sweep.json]

For each workload: median device time of `reps` dg_apply calls (CUDA events, after 3
warm-ups), DOFs/s, the paper's model GFLOP/s (FLOPDOF x DOFs/s), and the
volume-only variant (terms = DG_VOLUME) for the C4 rows, as SURVEY.md 8(a)/(d) asks.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1711_10885_b200 import configs, dg, perfmodel  # noqa: E402


def time_apply(op, z, y, terms, reps):
    for _ in range(3):
        op.apply(z, y, terms=terms)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply(z, y, terms=terms)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def run(cfg, reps, volume_only):
    op = dg.from_config(cfg)
    z = torch.empty(op.ndofs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(z)
    op.fill_uniform_local(z, cfg.seed)
    t, tmin = time_apply(op, z, y, dg.ALL, reps)
    row = {"config": cfg.name, "k": cfg.k, "ncells": list(cfg.ncells), "ndofs": cfg.ndofs, "ms": t * 1e3,
           "ms_min": tmin * 1e3, "gdofs": cfg.ndofs / t / 1e9,
           "model_flop_per_dof": perfmodel.flopdof(3, cfg.k),
           "model_gflops": perfmodel.flopdof(3, cfg.k) * cfg.ndofs / t / 1e9,
           "kernel": op.kernel_info()}
    if volume_only:
        tv, _ = time_apply(op, z, y, dg.VOLUME, reps)
        row.update({"vol_ms": tv * 1e3, "vol_gdofs": cfg.ndofs / tv / 1e9,
                    "vol_model_gflops": perfmodel.flopdof_vol(3, cfg.k) * cfg.ndofs / tv / 1e9})
    op.close()
    del z, y
    torch.cuda.empty_cache()
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    ap.add_argument("--skip-c5", action="store_true")
    a = ap.parse_args()
    rows = []
    for k in range(1, 11):
        rows.append(run(configs.c4(k), a.reps, True))
        print(json.dumps(rows[-1]), flush=True)
    for cfg in [configs.c2(), configs.c3()] + ([] if a.skip_c5 else [configs.c5_weak(1), configs.c5_strong()]):
        rows.append(run(cfg, a.reps, False))
        print(json.dumps(rows[-1]), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
