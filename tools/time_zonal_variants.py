"""Headline zonal compress passes (adct_compress_psnr, SSE only) at each of C5's r for several
library variants (paths to libadct_*.so, 'default' = in-tree): per-r HBM fraction (1 B/px) on N
C5-kind 4096^2 images, best of 3 x 3 launches; SSE compared against the first variant.

    python tools/time_zonal_variants.py default tune_variants/libadct_x.so ...   (N via IMAGES)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, torch
sys.path.insert(0, __ROOT__)
from paper_1402_6034_b200 import _lib
if __LIBV__ != "default":
    _lib.LIB_PATH = __LIBV__
    # older builds may lack newer entries: bind only what the timing uses
    _lib.SIGNATURES = {k: v for k, v in _lib.SIGNATURES.items()
                       if k in ("adct_compress_psnr", "adct_psnr", "adct_status_string", "adct_last_cuda_error")}
import paper_1402_6034_b200 as A
from synth import images as S
RS = (1, 3, 6, 10, 15, 21, 28, 36)
x = S.device_mixed(__N__, 4096, 4096, device="cuda")
sse = torch.empty((8, x.shape[0]), dtype=torch.float64, device="cuda")
def best(fn):
    fn(); torch.cuda.synchronize(); b = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): fn()
        e1.record(); torch.cuda.synchronize(); b = min(b, e0.elapsed_time(e1) / 3)
    return b
ms = {}
for k, r in enumerate(RS):
    ms[str(r)] = best(lambda: A.compress_psnr(x, r, sse=sse[k]))
out = sse.cpu().flatten().tolist()
print(json.dumps({"lib": __LIBV__, "ms": ms, "px": x.numel(), "sse": out}))
'''


def main():
    n = os.environ.get("IMAGES", "128")
    res = []
    for lib in sys.argv[1:]:
        code = CHILD.replace("__ROOT__", repr(ROOT)).replace("__LIBV__", repr(lib)).replace("__N__", n)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        if r.returncode:
            print(lib, "FAILED", r.stderr[-1500:])
            continue
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    for d in res:
        rel = max(abs(a - b) / max(abs(b), 1e-30) for a, b in zip(d["sse"], res[0]["sse"]))
        fr = {r: d["px"] / (v * 1e-3) / 1e9 / peak for r, v in d["ms"].items()}
        tot = len(fr) / sum(1 / f for f in fr.values())
        print(f"{os.path.basename(d['lib']):22s} step-equivalent frac {tot:.4f} | " +
              " ".join(f"r{r}:{f:.3f}" for r, f in fr.items()) + f" | max rel SSE vs first {rel:.1e}")


if __name__ == "__main__":
    main()
