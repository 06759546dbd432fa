"""Build libdg_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1711_10885_b200.build [--force] [-v]

One object per basis size n = k+1 (dg_cell_inst.cu with -DDG_N=n) plus the host ABI,
tables, dispatch, NCCL loader and auxiliary kernels; objects compile in parallel.
"""
import argparse
import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libdg_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
NS = list(range(2, 12))


# (n, m) pairs of the variable-velocity / over-integrated kernel: m = n (q = 2p), m = n + 2
# (q = 2p + 4, the paper's Taylor-Green run) and ceil((3k + 5) / 2) (q = 3p + 4), m <= 16
VB = sorted({(n, m) for n in range(2, 12) for m in (n, n + 2, -(-(3 * n + 2) // 2)) if m <= 16})
# (n, m) pairs of the multilinear-geometry kernel: m = n, n + 2 and ceil((3k + 5) / 2) (q = 3p + 4,
# PAPER.md:957-961), m <= 16 (the cell's shared memory)
GEO = sorted({(n, m) for n in range(2, 12) for m in (n, n + 2, -(-(3 * n + 2) // 2)) if m <= 16})


def _sources():
    jobs = []
    for n in NS:
        jobs.append((os.path.join(CSRC, "dg_cell_inst.cu"), os.path.join(OBJ, "dg_cell_n%d.o" % n), ["-DDG_N=%d" % n]))
    for n, m in VB:
        jobs.append((os.path.join(CSRC, "dg_vb_inst.cu"), os.path.join(OBJ, "dg_vb_n%d_m%d.o" % (n, m)),
                     ["-DDG_N=%d" % n, "-DDG_M=%d" % m]))
    for n, m in GEO:
        jobs.append((os.path.join(CSRC, "dg_geo_inst.cu"), os.path.join(OBJ, "dg_geo_n%d_m%d.o" % (n, m)),
                     ["-DDG_N=%d" % n, "-DDG_M=%d" % m]))
    for name in ("dg_aux.cu", "dg_matrix.cu", "dg_abi.cpp", "dg_dispatch.cpp", "dg_nccl.cpp", "dg_fabric.cpp", "dg_p2p.cpp", "tables.cpp"):
        base = os.path.splitext(name)[0]
        extra = ["-x", "cu"] if name.endswith(".cpp") else []
        jobs.append((os.path.join(CSRC, name), os.path.join(OBJ, base + ".o"), extra))
    return jobs


# the sources each kernel family's translation unit compiles (its .cu, the headers it includes, the
# shared declarations and the tables it is given)
KERNEL_SOURCES = {
    "cell": ["dg_cell_inst.cu", "dg_cell.cuh", "dg_reg.cuh", "dg_mma8.cuh", "dg_internal.h", "tables.cpp"],
    "gen": ["dg_cell_inst.cu", "dg_gen.cuh", "dg_cell.cuh", "dg_reg.cuh", "dg_internal.h", "tables.cpp"],
    "vb": ["dg_vb_inst.cu", "dg_vb.cuh", "dg_cell.cuh", "dg_internal.h", "tables.cpp"],
    "geo": ["dg_geo_inst.cu", "dg_geo.cuh", "dg_cell.cuh", "dg_internal.h", "tables.cpp"],
}


def kernel_family(kernel_name):
    """'cell' | 'gen' | 'vb' | 'geo' for a kernel name such as 'dg_gen_kernel<8>'."""
    for fam in ("gen", "vb", "geo"):
        if "dg_%s" % fam in kernel_name:
            return fam
    return "cell"


def kernel_hash(family="cell"):
    """Hash of everything that determines one kernel family's compiled code (its translation unit
    and the headers it includes, the tables, the flags): the key under which
    profiles/ncu_full_summary.json stores executed-flop counts, so bench.py never pairs a timing
    with the counts of another build. Host-only files (the ABI, dispatch, transport) are not in it."""
    h = hashlib.sha256()
    h.update(" ".join(ARCH + FLAGS[:3]).encode())
    for f in KERNEL_SOURCES[family]:
        h.update(f.encode())
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "dg.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, ptxas_v=False):
    os.makedirs(OBJ, exist_ok=True)
    deps = _deps()
    jobs = _sources()

    def compile_one(job):
        src, obj, extra = job
        if not force and not _stale(obj, deps):
            return obj, ""
        cmd = [NVCC] + ARCH + FLAGS + extra + (["-Xptxas", "-v"] if ptxas_v else []) + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (" ".join(cmd), r.stdout, r.stderr))
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        results = list(ex.map(compile_one, jobs))
    if verbose:
        for obj, log in results:
            if log:
                print(os.path.basename(obj), log, file=sys.stderr)
    objs = [o for o, _ in results]
    if force or _stale(LIB, objs):
        tmp = LIB + ".tmp%d" % os.getpid()
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--ptxas", action="store_true", help="print -Xptxas -v (registers, spills)")
    a = ap.parse_args()
    print(build(force=a.force or a.ptxas, verbose=a.verbose or a.ptxas, ptxas_v=a.ptxas))
