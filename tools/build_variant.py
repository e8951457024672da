"""Build a tuning variant of libadct.so with extra -D flags (measurement only, not the product):

    python tools/build_variant.py NAME [--tu adct_api] -DADCT_MINB_QRES=3 ...

recompiles the listed translation units (default: all) with the flags, reuses build/obj/*.o for the
rest, and links tune_variants/libadct_NAME.so (git-ignored; travels with gpurun).  tools/time_quant_variants.py loads such a library
by pointing paper_1402_6034_b200._lib.LIB_PATH at it before the first call."""
import argparse
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1402_6034_b200 import build as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("name")
ap.add_argument("--tu", action="append", default=None)
a, defs = ap.parse_known_args()
B.build()
out = os.path.join(B.ROOT, "tune_variants", a.name)
os.makedirs(out, exist_ok=True)
import concurrent.futures as cf  # noqa: E402


def one(src):
    tu = os.path.basename(src)[:-3]
    if a.tu is None or tu in a.tu:
        obj = os.path.join(out, tu + ".o")
        cmd = [B.nvcc()] + B.ARCH + B.NVFLAGS + defs + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        open(obj + ".log", "w").write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(r.stderr[-3000:])
        return obj
    return os.path.join(B.BUILD, tu + ".o")


with cf.ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, B._sources()))
lib = os.path.join(B.ROOT, "tune_variants", f"libadct_{a.name}.so")
subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", lib] + objs, check=True)
print(lib)
