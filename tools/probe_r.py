"""Compile single compress-kernel instantiations and print the static register-read estimate
(tools/sass_regread.py) — the CPU-side loop for kernel-body experiments (no GPU needed).

    python tools/probe_r.py --r 10,21,36 [-DADCT_X=1 ...] [--keep DIR]
"""
import argparse
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_1402_6034_b200 import build as B  # noqa: E402
import sass_regread as SR  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--r", default="10,21,36")
ap.add_argument("--keep", default=None)
ap.add_argument("--quant", action="store_true", help="probe k_compress<64, QUANT> instead")
a, defs = ap.parse_known_args()
rs = [int(v) for v in a.r.split(",")]
d = a.keep or tempfile.mkdtemp(prefix="probe_")
os.makedirs(d, exist_ok=True)


def one(r):
    src = os.path.join(d, f"probe_{r}.cu")
    kind = "MODE_QUANT" if a.quant else "MODE_ZONAL"
    with open(src, "w") as f:
        f.write('#include "adct_kernels.cuh"\nnamespace adct {\n'
                f'CompressKernel probe_{r}() {{ return &k_compress<{r}, {kind}, REC_NONE>; }}\n}}\n')
    obj = src[:-3] + ".o"
    cmd = [B.nvcc()] + B.ARCH + B.NVFLAGS + defs + ["-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode:
        sys.exit(res.stderr[-3000:])
    regs = [ln for ln in res.stderr.split("\n") if "registers" in ln]
    return obj, (regs[-1].strip() if regs else "")


import concurrent.futures as cf  # noqa: E402
with cf.ThreadPoolExecutor(len(rs)) as ex:
    outs = list(ex.map(one, rs))
for r, (obj, regs) in zip(rs, outs):
    res = SR.analyse([obj], {r}, mode=1 if a.quant else 0)
    n, c = res[r]
    cnt, cyc = SR.breakdown(obj, r)
    top = ", ".join(f"{k} {cnt[k]}/{cyc[k]}" for k, _ in cyc.most_common(7))
    print(f"r={r:2d} instr {n:4d} read-cycles {c:5d} bound@670 {670 / max(n, c):.3f} | {top} | {regs[-60:]}")
