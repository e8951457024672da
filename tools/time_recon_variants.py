"""Fused compress with a reconstruction output (32 x 4096^2 C5-kind images): zonal r = 10 / 36 with
f32 (5 B/px) and u8 (2 B/px) reconstruction, quantiser q = 16 with u8, for several library variants
(paths to libadct_*.so, 'default' = in-tree); outputs compared against the first variant.

    python tools/time_recon_variants.py default tune_variants/libadct_rec_old.so ..."""
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
import paper_1402_6034_b200 as A
from synth import images as S
x = S.device_mixed(32, 4096, 4096, seed=0, device="cuda")
sse = torch.empty(32, dtype=torch.float64, device="cuda")
rf = torch.empty((32, 4096, 4096), dtype=torch.float32, device="cuda")
ru = torch.empty((32, 4096, 4096), dtype=torch.uint8, device="cuda")
def best(fn):
    fn(); torch.cuda.synchronize(); b = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize(); b = min(b, e0.elapsed_time(e1) / 5)
    return b
ms = {}
ck = []
for name, r, q, kind, out in (("z10f32", 10, 0.0, "f32", rf), ("z10u8", 10, 0.0, "u8", ru), ("z36f32", 36, 0.0, "f32", rf),
                              ("z36u8", 36, 0.0, "u8", ru), ("q16u8", 64, 16.0, "u8", ru)):
    ms[name] = best(lambda: A.compress_psnr(x, r, q=q, sse=sse, recon=kind, recon_out=out))
    A.compress_psnr(x, r, q=q, sse=sse, recon=kind, recon_out=out)
    ck.append(float(out.double().sum().item()) if kind == "f32" else int(out.to(torch.int64).sum().item()))
    ck.append(round(float(sse.sum().item()), 3))
print(json.dumps({"lib": __LIBV__, "ms": ms, "ck": ck}))
'''


def main():
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    res = []
    for lib in sys.argv[1:]:
        code = CHILD.replace("__ROOT__", repr(ROOT)).replace("__LIBV__", repr(lib))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        if r.returncode:
            print(lib, "FAILED", r.stderr[-1500:])
            continue
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    px = 32 * 4096 * 4096
    bpp = {"z10f32": 5, "z10u8": 2, "z36f32": 5, "z36u8": 2, "q16u8": 2}
    for d in res:
        parts = " | ".join(f"{k} {v:.3f} ms {px / (v * 1e-3) / 1e9:.0f} Gpix/s frac {bpp[k] * px / (v * 1e-3) / 1e9 / peak:.3f}"
                           for k, v in d["ms"].items())
        print(f"{os.path.basename(d['lib']):20s} {parts} | output {'identical' if d['ck'] == res[0]['ck'] else 'DIFFERENT'}")


if __name__ == "__main__":
    main()
