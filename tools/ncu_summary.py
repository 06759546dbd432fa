"""Summarise an ncu --set full report of the cell kernel (read here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--name C3] [--ndofs N] [--json out.json] [--md out.md]

Prints the numbers the roofline/traffic claims rest on: duration, DRAM bytes per
launch, FP64 pipe utilisation, executed FP64 flops, shared-memory wavefronts and
bank conflicts, occupancy, issue-slot use and the top stall reasons.
"""
import argparse
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dfma_per_cycle": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
    "dadd_per_cycle": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
    "dmul_per_cycle": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed",
    "dfma_sum": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "dadd_sum": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dmul_sum": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "cycles": "sm__cycles_elapsed.avg",
    "clock_hz": "sm__cycles_elapsed.avg.per_second",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}
UNITS_TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TIME_TO_NS = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}
FREQ = {"hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        launches.append(d)
    return launches


def num(d, key):
    if key not in d:
        return None
    v, u = d[key]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    if u in UNITS_TO_BYTES:
        x *= UNITS_TO_BYTES[u]
    if u in TIME_TO_NS:
        x *= TIME_TO_NS[u]
    if u in FREQ:
        x *= FREQ[u]
    return x


def summarize(d):
    s = {k: num(d, m) for k, m in KEYS.items()}
    s["kernel"] = d.get("Kernel Name", ("?", ""))[0]
    if s["dram_read"] is not None and s["dram_write"] is not None:
        s["dram_bytes_per_launch"] = s["dram_read"] + s["dram_write"]
    cyc = s.get("cycles")
    if s.get("dfma_sum") is not None:       # thread-level FP64 instruction counts (flops = 2 DFMA + DADD + DMUL)
        s["executed_fp64_flops"] = 2 * s["dfma_sum"] + (s.get("dadd_sum") or 0) + (s.get("dmul_sum") or 0)
    elif cyc and s.get("dfma_per_cycle") is not None:
        s["executed_fp64_flops"] = cyc * (2 * s["dfma_per_cycle"] + (s.get("dadd_per_cycle") or 0)
                                          + (s.get("dmul_per_cycle") or 0))
    stalls = []
    for h, (v, u) in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    s["top_stalls"] = [(n, round(v, 3)) for v, n in sorted(stalls, reverse=True)[:8]]
    return s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--name", default=None)
    ap.add_argument("--ndofs", type=int, default=None)
    ap.add_argument("--json", default=None, help="merge {name: summary} into this JSON file")
    ap.add_argument("--kernel", default=None, help="substring of the kernel name to summarise")
    args = ap.parse_args()
    launches = raw(args.rep)
    keys = (args.kernel,) if args.kernel else ("dg_cell", "dg_reg", "dg_gen", "dg_vb", "dg_geo")
    cell = [d for d in launches if any(k in d.get("Kernel Name", ("", ""))[0] for k in keys)] or launches
    s = summarize(cell[0])
    sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
    from paper_1711_10885_b200.build import kernel_family, kernel_hash
    s["build_hash"] = kernel_hash(kernel_family(s["kernel"]))   # the build this capture belongs to (bench.py checks it)
    if args.ndofs:
        s["ndofs"] = args.ndofs
        if s.get("executed_fp64_flops"):
            s["executed_flops_per_dof"] = s["executed_fp64_flops"] / args.ndofs
        if s.get("dram_bytes_per_launch"):
            s["dram_bytes_per_dof"] = s["dram_bytes_per_launch"] / args.ndofs
    print(json.dumps(s, indent=1))
    if args.json and args.name:
        try:
            with open(args.json) as f:
                allj = json.load(f)
        except Exception:
            allj = {}
        allj[args.name] = s
        with open(args.json, "w") as f:
            json.dump(allj, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())
