"""Split a kernel's SASS (ncu --page source --print-source sass of a --set full report) at its
CTA barriers and sum the warp-stall samples and executed instructions per segment: where the
time goes phase by phase (the kernels are straight-line code between barriers).

    python tools/ncu_phases.py gpurun_out/a-k7_full.ncu-rep
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(rep, split="BAR.SYNC"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    lines = out.splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[i:]))))
    hdr = rows[0]
    cs = hdr.index("Warp Stall Sampling (All Samples)")
    ci = hdr.index("Instructions Executed")
    stall_cols = [k for k, h in enumerate(hdr) if h.startswith("stall_")]
    segs, cur = [], None
    total = 0
    for r in rows[1:]:
        if len(r) <= ci:
            continue
        src = r[1].strip()
        if cur is None:
            cur = {"first": src, "samples": 0, "inst": 0, "n": 0, "ops": Counter(), "stalls": Counter()}
        s = int(r[cs] or 0)
        cur["samples"] += s
        total += s
        cur["inst"] += int(r[ci] or 0)
        cur["n"] += 1
        op = src.split()[0] if src else ""
        if op.startswith("@"):
            op = src.split()[1]
        cur["ops"][op.split(".")[0]] += int(r[ci] or 0)
        for k in stall_cols:
            v = r[k]
            if v and v not in ("-", "0"):
                cur["stalls"][hdr[k][6:]] += int(v)
        if split in src:
            segs.append(cur)
            cur = None
    if cur:
        segs.append(cur)
    for k, sg in enumerate(segs):
        top = ", ".join(f"{o}:{c / max(1, sg['inst']) * 100:.0f}%" for o, c in sg["ops"].most_common(5))
        st = ", ".join(f"{o}:{c / max(1, sg['samples']) * 100:.0f}%" for o, c in sg["stalls"].most_common(4))
        print(f"seg {k:2d}: {sg['samples'] / max(1, total) * 100:5.1f}% samples  {sg['inst'] / 1e6:9.1f}M warp-inst  "
              f"{sg['n']:5d} sass | {top} | {st}")


if __name__ == "__main__":
    main(*sys.argv[1:])
