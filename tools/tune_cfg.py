"""Build launch-configuration variants of one degree's cell kernel (CPU side).

    python tools/tune_cfg.py N TPC,P,C,MINB [TPC,P,C,MINB ...]

Each variant recompiles only dg_cell_inst.cu for that n (with -DDG_TPC/-DDG_P/-DDG_C/
-DDG_MINB) and relinks it with the standard objects into variants/n<N>_<tpc>_<p>_<c>_<mb>.so,
selectable at run time with DG_LIB=... (paper_1711_10885_b200/dg.py).
"""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_10885_b200 import build as B  # noqa: E402


def variant(n, tpc, p, c, mb):
    name = "n%d_%d_%d_%d_%d" % (n, tpc, p, c, mb)
    obj = os.path.join(ROOT, "build", "var", name + ".o")
    os.makedirs(os.path.dirname(obj), exist_ok=True)
    cmd = [B.NVCC] + B.ARCH + B.FLAGS + ["-DDG_N=%d" % n, "-DDG_TPC=%d" % tpc, "-DDG_P=%d" % p, "-DDG_C=%d" % c,
                                         "-DDG_MINB=%d" % mb, "-Xptxas", "-v", "-c",
                                         os.path.join(B.CSRC, "dg_cell_inst.cu"), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        return name, "compile failed: " + r.stderr[-400:]
    info = [l.strip() for l in r.stderr.splitlines() if "Used" in l or "spill" in l]
    objs = [os.path.join(B.OBJ, f) for f in sorted(os.listdir(B.OBJ)) if f.endswith(".o") and f != "dg_cell_n%d.o" % n]
    out = os.path.join(ROOT, "variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    r = subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", out, obj] + objs + ["-ldl", "-lpthread"],
                       capture_output=True, text=True)
    if r.returncode:
        return name, "link failed: " + r.stderr[-400:]
    return name, " | ".join(info[-2:])


def main():
    B.build()
    n = int(sys.argv[1])
    specs = [tuple(int(x) for x in a.split(",")) for a in sys.argv[2:]]
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for name, info in ex.map(lambda s: variant(n, *s), specs):
            print(name, info)


if __name__ == "__main__":
    main()
