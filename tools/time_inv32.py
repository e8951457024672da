import sys, torch
sys.path.insert(0, "/root/repo")
import paper_1402_6034_b200 as A
from synth import images as S
import json
peak = json.load(open("/root/repo/MEASURED_PEAKS.json"))["hbm_gbs"]
x = S.device_mixed(16, 4096, 4096, seed=0, device="cuda")
c32 = A.forward(x, coef="i32"); cf = A.forward(x, coef="f32")
rf = torch.empty((16, 4096, 4096), dtype=torch.float32, device="cuda")
ru = torch.empty((16, 4096, 4096), dtype=torch.uint8, device="cuda")
def best(fn):
    fn(); torch.cuda.synchronize(); b = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize(); b = min(b, e0.elapsed_time(e1) / 5)
    return b
px = x.numel()
for name, c, out, dst, bpp in (("i32->f32", c32, "f32", rf, 8), ("i32->u8", c32, "u8", ru, 5), ("f32->f32", cf, "f32", rf, 8), ("f32->u8", cf, "u8", ru, 5)):
    ms = best(lambda: A.inverse(c, r=64, out=out, dst=dst))
    print(f"inverse {name}: {ms:.3f} ms frac {bpp * px / (ms * 1e-3) / 1e9 / peak:.3f}")
