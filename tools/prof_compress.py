"""Small driver for ncu captures: compress at the given r values (and forward-only) on n C5 images."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_6034_b200 as A
from synth import images as S

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--r", type=str, default="1,36")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--fwd", action="store_true")
ap.add_argument("--quant", action="store_true")
a = ap.parse_args()
x = S.device_mixed(a.n, 4096, 4096, device="cuda")
sse = torch.empty(a.n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for _ in range(a.reps):
    for r in [int(v) for v in a.r.split(",") if v]:
        A.compress_psnr(x, r, sse=sse)
    if a.quant:
        A.compress_psnr(x, 64, q=16.0, sse=sse)
    if a.fwd:
        out = torch.empty((a.n, 4096, 4096), dtype=torch.int16, device="cuda")
        A.forward(x, out=out)
torch.cuda.synchronize()
print("ok")
