"""Build the bounds-checked library (-DDG_CHECK: device-side index asserts that trap) into
variants/checked/libdg_b200.so (travels with gpurun); run the GPU tests against it with
DG_LIB=$PWD/variants/checked/libdg_b200.so."""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_10885_b200 import build as B  # noqa: E402


def main():
    out = os.path.join(ROOT, "variants", "checked")
    os.makedirs(out, exist_ok=True)

    def one(job):
        src, obj, extra = job
        o = os.path.join(out, os.path.basename(obj))
        subprocess.check_call([B.NVCC] + B.ARCH + B.FLAGS + ["-DDG_CHECK"] + extra + ["-c", src, "-o", o])
        return o

    with cf.ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(one, B._sources()))
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", os.path.join(out, "libdg_b200.so")] + objs +
                          ["-ldl", "-lpthread"])
    print(os.path.join(out, "libdg_b200.so"))


if __name__ == "__main__":
    main()
