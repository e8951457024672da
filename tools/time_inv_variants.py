"""Standalone inverse from an int16 coefficient plane (32 x 4096^2, C5-kind images) to f32 (6 B/px)
and to u8 (3 B/px) for several library variants (paths to libadct_*.so, 'default' = in-tree):
ms, GB/s, HBM fraction; outputs compared against the first variant.  Best of 3 x 10 launches.

    python tools/time_inv_variants.py default tune_variants/libadct_inv_old.so ..."""
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
coef = A.forward(x)
del x
rf = torch.empty((32, 4096, 4096), dtype=torch.float32, device="cuda")
ru = torch.empty((32, 4096, 4096), dtype=torch.uint8, device="cuda")
def best(fn):
    fn(); torch.cuda.synchronize(); b = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): fn()
        e1.record(); torch.cuda.synchronize(); b = min(b, e0.elapsed_time(e1) / 10)
    return b
msf = best(lambda: A.inverse(coef, r=64, out="f32", dst=rf))
msu = best(lambda: A.inverse(coef, r=10, out="u8", dst=ru))
A.inverse(coef, r=10, out="f32", dst=rf)
ck = [float(rf.double().sum().item()), float(rf[:, ::7, ::5].double().pow(2).sum().item()), int(ru.to(torch.int64).sum().item())]
print(json.dumps({"lib": __LIBV__, "msf": msf, "msu": msu, "ck": ck}))
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
    for d in res:
        gf = 6 * px / (d["msf"] * 1e-3) / 1e9
        gu = 3 * px / (d["msu"] * 1e-3) / 1e9
        print(f"{os.path.basename(d['lib']):22s} inverse i16->f32: {d['msf']:.3f} ms {gf:.0f} GB/s frac {gf / peak:.3f} | "
              f"i16->u8: {d['msu']:.3f} ms {gu:.0f} GB/s frac {gu / peak:.3f} | "
              f"output {'identical' if d['ck'] == res[0]['ck'] else 'DIFFERENT ' + str(d['ck'])}")


if __name__ == "__main__":
    main()
