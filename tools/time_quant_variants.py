"""Time C4-shaped quantiser compress (SSE only, q = 16) and a zonal r for each library variant
given on the command line (paths to libadct_*.so; 'default' = the in-tree build).  Best of 3 x 5
launches with CUDA events; also checks every variant's SSE equals the default build's.

    python tools/time_quant_variants.py default tune_variants/libadct_q3.so ...
"""
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
v = S.device_video(NFR, 4320, 7680, seed=0, device="cuda")
sse = torch.empty(NFR, dtype=torch.float64, device="cuda")
def best(fn):
    fn(); torch.cuda.synchronize(); b = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize(); b = min(b, e0.elapsed_time(e1) / 5)
    return b
ms = best(lambda: A.compress_psnr(v, 64, q=16.0, sse=sse))
out = A.compress_psnr(v, 64, q=16.0).cpu().tolist()[:8]
print(json.dumps({"lib": __LIBV__, "ms": ms, "gpix_s": v.numel() / ms / 1e6, "sse": out}))
'''


def main():
    import json
    peak = 6542.4
    res = []
    for lib in sys.argv[1:]:
        code = CHILD.replace("__ROOT__", repr(ROOT)).replace("__LIBV__", repr(lib)).replace("NFR", os.environ.get("FRAMES", "8"))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        if r.returncode:
            print(lib, "FAILED", r.stderr[-2000:])
            continue
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    base = res[0]["sse"] if res else None
    for d in res:
        rel = max(abs(a - b) / max(abs(b), 1e-30) for a, b in zip(d["sse"], base))
        print(f"{os.path.basename(d['lib']):24s} C4 quant q=16: {d['ms']:.3f} ms  {d['gpix_s']:.0f} Gpix/s  "
              f"HBM frac {d['gpix_s'] / peak:.3f}  max rel SSE vs first {rel:.1e}")


if __name__ == "__main__":
    main()
