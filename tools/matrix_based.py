"""Matrix-based comparison (Table 1's matrix-based columns).

    python tools/matrix_based.py [--ks 1,2,...,10] [--reps 10] [--budget 24e9] [--big] [--out FILE]

Per degree k, on Problem A scaled down so that the assembled block-stencil matrix fits in
`budget` bytes (configs.problem_a_matrix: periodic, per-cell SPD tensors):
  - assembly time of dg_assemble (probing the fused sum-factorized kernel), as DOFs/s;
  - dg_matrix_apply: median device time of `reps` calls (CUDA events), DOFs/s and HBM GB/s of the
    algorithmic traffic (perfmodel.matrix_bytes_per_dof), parity against the matrix-free apply;
  - the matrix-free dg_apply on the same mesh, and (--big) on the full Problem A mesh (~4e8 DOFs,
    configs.problem_a), whose rate the paper divides by the matrix-based one ("A / matrix-based").
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_10885_b200 import configs, dg, perfmodel  # noqa: E402


def dg_matrix_gb(cfg, k):
    n3 = (k + 1) ** 3
    return cfg.ndofs * 7 * (n3 + (n3 & 1)) * 8 / 1e9


def median_ms(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def matrix_free_rate(cfg, reps):
    op = dg.from_config(cfg)
    op.set_tensor_field(cfg.dfield_seed)
    z = torch.empty(cfg.ndofs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(z)
    op.fill_uniform_local(z, cfg.seed)
    ms, _ = median_ms(lambda: op.apply(z, y), reps)
    op.close()
    return cfg.ndofs / (ms * 1e-3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ks", default="1,2,3,4,5,6,7,8,9,10")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--budget", type=float, default=24e9)
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for k in [int(v) for v in a.ks.split(",")]:
        cfg = configs.problem_a_matrix(k, a.budget)
        op = dg.from_config(cfg)
        op.set_tensor_field(cfg.dfield_seed)
        z = torch.empty(cfg.ndofs, dtype=torch.float64, device="cuda")
        op.fill_uniform_local(z, cfg.seed)
        y = torch.empty_like(z)
        ymf = torch.empty_like(z)
        A = torch.empty(op.matrix_size(), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op.assemble(A)
        torch.cuda.synchronize()
        t_asm = time.perf_counter() - t0
        mb_ms, mb_min = median_ms(lambda: op.matrix_apply(A, z, y), a.reps)
        mf_ms, _ = median_ms(lambda: op.apply(z, ymf), a.reps)
        torch.cuda.synchronize()
        err = float((y - ymf).abs().max() / ymf.abs().max())
        op.close()
        del A
        torch.cuda.empty_cache()
        bpd = perfmodel.matrix_bytes_per_dof(k)
        row = {"k": k, "config": cfg.name, "ncells": list(cfg.ncells), "ndofs": cfg.ndofs,
               "matrix_gb": dg_matrix_gb(cfg, k),
               "assembly_s": t_asm, "assembly_mdofs": cfg.ndofs / t_asm / 1e6,
               "matrix_apply_ms": mb_ms, "matrix_apply_ms_min": mb_min,
               "matrix_apply_mdofs": cfg.ndofs / (mb_ms * 1e-3) / 1e6,
               "matrix_apply_hbm_gbs": cfg.ndofs * bpd / (mb_ms * 1e-3) / 1e9, "bytes_per_dof": bpd,
               "matrix_free_same_mesh_mdofs": cfg.ndofs / (mf_ms * 1e-3) / 1e6,
               "parity_matrix_vs_matrix_free": err,
               "paper_matrix_mdofs": perfmodel.PAPER_TABLE1_MATRIX_MDOFS.get(k),
               "paper_assembly_mdofs": perfmodel.PAPER_TABLE1_ASSEMBLY_MDOFS.get(k),
               "paper_matrix_free_A_mdofs": perfmodel.PAPER_TABLE1_A_MDOFS.get(k)}
        if a.big:
            row["matrix_free_problem_a_mdofs"] = matrix_free_rate(configs.problem_a(k), a.reps) / 1e6
            row["ratio_matrix_free_A_over_matrix"] = row["matrix_free_problem_a_mdofs"] / row["matrix_apply_mdofs"]
        pm = perfmodel.PAPER_TABLE1_MATRIX_MDOFS.get(k)
        if pm:
            row["paper_ratio_A_over_matrix"] = perfmodel.PAPER_TABLE1_A_MDOFS[k] / pm
        print(json.dumps(row), flush=True)
        rows.append(row)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
