"""Diagnostic: compress throughput per r on 256 x 4096^2 (4 GiB) and forward-only."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_6034_b200 as A
from synth import images as S

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

n, h, w = 256, 4096, 4096
G = n * h * w
x = S.device_mixed(n, h, w, device="cuda")
sse = torch.empty(n, dtype=torch.float64, device="cuda")
for r in list(range(1, 65, 1)) if "all" in sys.argv else (1, 3, 6, 10, 15, 21, 28, 36, 64):
    ms = t(lambda: A.compress_psnr(x, r, sse=sse))
    print(f"r={r:2d} {ms:7.3f} ms {G/ms/1e6:7.0f} GB/s  frac={G/ms/1e6/6534.1:.3f}", flush=True)
ms = t(lambda: A.compress_psnr(x, 64, q=16.0, sse=sse))
print(f"quant q=16 {ms:7.3f} ms {G/ms/1e6:7.0f} GB/s frac={G/ms/1e6/6534.1:.3f}")
out = torch.empty((n, h, w), dtype=torch.int16, device="cuda")
ms = t(lambda: A.forward(x, out=out))
print(f"fwd i16 {ms:7.3f} ms {3*G/ms/1e6:7.0f} GB/s frac={3*G/ms/1e6/6534.1:.3f}")
