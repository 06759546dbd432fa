"""Build the bounds-checked library (-DDG_CHECK: device-side index asserts that trap) into
checkbuild/libdg_b200.so; run the GPU tests against it with DG_LIB=$PWD/checkbuild/libdg_b200.so."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_10885_b200 import build as B  # noqa: E402


def main():
    out = os.path.join(ROOT, "checkbuild")
    os.makedirs(out, exist_ok=True)
    objs = []
    for src, obj, extra in B._sources():
        o = os.path.join(out, os.path.basename(obj))
        cmd = [B.NVCC] + B.ARCH + B.FLAGS + ["-DDG_CHECK"] + extra + ["-c", src, "-o", o]
        subprocess.check_call(cmd)
        objs.append(o)
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", os.path.join(out, "libdg_b200.so")] + objs +
                          ["-ldl", "-lpthread"])
    print(os.path.join(out, "libdg_b200.so"))


if __name__ == "__main__":
    main()
