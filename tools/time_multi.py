"""Fused multi-r sweep (adct_compress_psnr_multi, C5's r set) vs eight independent passes on
C5-kind images: Gpixel-passes/s and the per-r-pass HBM-equivalent fraction."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_6034_b200 as A
from synth import images as S

RS = (1, 3, 6, 10, 15, 21, 28, 36)


def best(fn, rounds=3, reps=3):
    fn(); torch.cuda.synchronize()
    b = 1e30
    for _ in range(rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record(); torch.cuda.synchronize(); b = min(b, e0.elapsed_time(e1) / reps)
    return b


x = S.device_mixed(int(sys.argv[1]) if len(sys.argv) > 1 else 128, 4096, 4096, device="cuda")
sse = torch.empty((len(RS), x.shape[0]), dtype=torch.float64, device="cuda")
pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
t_sep = best(lambda: [A.compress_psnr(x, r, sse=sse[k]) for k, r in enumerate(RS)])
t_mul = best(lambda: A.compress_psnr_multi(x, RS, sse=sse))
px = x.numel() * len(RS)
for name, t in (("8 independent passes", t_sep), ("fused multi-r", t_mul)):
    print(f"{name:22s} {t:8.3f} ms  {px / t / 1e6:8.1f} Gpixel-passes/s  {px / t / 1e6 / pk:.3f} of HBM per pass-equivalent")
