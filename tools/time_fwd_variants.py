"""C3 forward (8192 x 512^2 uniform u8 -> int16 Y, 3 B/px) for several library variants (paths to
libadct_*.so, 'default' = in-tree): ms, GB/s, HBM fraction; outputs compared bit for bit (checksum
of the int16 plane) against the first variant.  Best of 3 x 10 launches, CUDA events.

    python tools/time_fwd_variants.py default tune_variants/libadct_fwd_old.so ..."""
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
x = S.device_uniform(8192, 512, 512, seed=0, device="cuda")
out = torch.empty((8192, 512, 512), dtype=torch.int16, device="cuda")
def best(fn):
    fn(); torch.cuda.synchronize(); b = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): fn()
        e1.record(); torch.cuda.synchronize(); b = min(b, e0.elapsed_time(e1) / 10)
    return b
ms = best(lambda: A.forward(x, out=out))
o32 = torch.empty((4096, 512, 512), dtype=torch.int32, device="cuda")
of = torch.empty((4096, 512, 512), dtype=torch.float32, device="cuda")
ms32 = best(lambda: A.forward(x[:4096], coef="i32", out=o32))
msf = best(lambda: A.forward(x[:4096], coef="f32", out=of))
ck = [int(out.view(torch.int32).sum(dtype=torch.int64).item()), int(out[:, ::7, ::5].to(torch.int64).pow(2).sum().item())]
masked = A.forward(x[:64], r=10)
ck.append(int(masked.to(torch.int64).abs().sum().item()))
ck.append(int(o32[:, ::3, ::5].to(torch.int64).abs().sum().item()))
ck.append(float(of[:, ::3, ::5].double().abs().sum().item()))
print(json.dumps({"lib": __LIBV__, "ms": ms, "ms32": ms32, "msf": msf, "ck": ck}))
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
    px = 8192 * 512 * 512
    for d in res:
        gbs = 3 * px / (d["ms"] * 1e-3) / 1e9
        g32 = 5 * px / 2 / (d["ms32"] * 1e-3) / 1e9
        gf = 5 * px / 2 / (d["msf"] * 1e-3) / 1e9
        print(f"{os.path.basename(d['lib']):22s} C3 forward i16: {d['ms']:.3f} ms  {gbs:.0f} GB/s  frac {gbs / peak:.3f} | "
              f"i32 (4096 img): frac {g32 / peak:.3f} | f32: frac {gf / peak:.3f} | "
              f"output {'identical' if d['ck'] == res[0]['ck'] else 'DIFFERENT'}")


if __name__ == "__main__":
    main()
