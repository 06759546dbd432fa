"""Build an experiment variant of one degree's translation unit (development aid).

    python tools/variant.py NAME N [-DFLAG[=V] ...]
    python tools/variant.py NAME matrix [-DFLAG[=V] ...]
    python tools/variant.py NAME geo:N:M [-DFLAG[=V] ...]     (multilinear-geometry kernel (n, m))
    python tools/variant.py NAME vb:N:M [-DFLAG[=V] ...]      (variable-velocity kernel (n, m))

Recompiles dg_cell_inst.cu for n = N (or dg_matrix.cu) with the extra flags, links it with the standard
objects into variants/NAME.so (select at run time with DG_LIB=$PWD/variants/NAME.so).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_10885_b200 import build as B  # noqa: E402


def main():
    name, flags = sys.argv[1], sys.argv[3:]
    what = sys.argv[2]
    B.build()
    obj = os.path.join(ROOT, "build", "var", name + ".o")
    os.makedirs(os.path.dirname(obj), exist_ok=True)
    if what == "matrix":
        src, replaced, defs = os.path.join(B.CSRC, "dg_matrix.cu"), "dg_matrix.o", []
    elif what.startswith(("geo:", "vb:")):
        fam, n, m = what.split(":")
        src = os.path.join(B.CSRC, "dg_%s_inst.cu" % fam)
        replaced, defs = "dg_%s_n%s_m%s.o" % (fam, n, m), ["-DDG_N=%s" % n, "-DDG_M=%s" % m]
    else:
        src, replaced, defs = os.path.join(B.CSRC, "dg_cell_inst.cu"), "dg_cell_n%d.o" % int(what), ["-DDG_N=%s" % what]
    cmd = [B.NVCC] + B.ARCH + B.FLAGS + defs + flags + ["-Xptxas", "-v", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit("compile failed:\n" + r.stderr[-2000:])
    lines = r.stderr.splitlines()
    for i, l in enumerate(lines):
        if "Compiling" in l and ("_kernel" in l):
            kn = l.split("'")[1] if "'" in l else l
            print(name, kn[:48], " | ".join(x.strip()[-70:] for x in lines[i + 1:i + 4] if "Used" in x or "spill" in x))
    objs = [os.path.join(B.OBJ, f) for f in sorted(os.listdir(B.OBJ)) if f.endswith(".o") and f != replaced]
    out = os.path.join(ROOT, "variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    r = subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", out, obj] + objs + ["-ldl", "-lpthread"],
                       capture_output=True, text=True)
    if r.returncode:
        sys.exit("link failed:\n" + r.stderr[-2000:])


if __name__ == "__main__":
    main()
