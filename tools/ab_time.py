"""A/B device timing of builds of the package on the same box (development aid).

    python tools/ab_time.py --trees . variants/r1 --workloads c3 a-k7 [--rounds 3]

Each tree is a directory holding a built paper_1711_10885_b200 package (or a variant .so of
tools/variant.py, loaded through DG_LIB with this tree's binding) (binding + .so; e.g. an
older commit's package copied under variants/, git-ignored). Runs tools/quick_time.py once per
(round, workload, tree) in a fresh process with PYTHONPATH at the tree, alternating the order so
clock drift hits all alike, and prints the median GDOF/s per (workload, tree)."""
import argparse
import os
import re
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trees", nargs="+", required=True)
    ap.add_argument("--workloads", nargs="+", default=["c3"])
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    res = {}
    for r in range(a.rounds):
        for w in a.workloads:
            for lib in (a.trees if r % 2 == 0 else a.trees[::-1]):
                if lib.endswith(".so"):       # a variant library (tools/variant.py) with this tree's binding
                    env = dict(os.environ, PYTHONPATH=ROOT, DG_LIB=os.path.abspath(lib))
                else:
                    env = dict(os.environ, PYTHONPATH=os.path.abspath(lib))
                    env.pop("DG_LIB", None)
                out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "quick_time.py"), w, str(a.reps)],
                                     capture_output=True, text=True, env=env).stdout
                m = re.search(r"GDOF/s ([0-9.]+)", out)
                res.setdefault((w, lib), []).append(float(m.group(1)) if m else float("nan"))
    for (w, lib), v in sorted(res.items()):
        print("%-10s %-50s median %.2f GDOF/s  runs %s" % (w, lib, statistics.median(v), " ".join("%.2f" % x for x in v)))


if __name__ == "__main__":
    main()
