"""Diagnostic: compress / forward throughput vs image geometry (same bytes)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_6034_b200 as A

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

G = 4 << 30
for (h, w) in [(4096, 4096), (512, 512), (512, 4096), (4096, 512), (16, 4096), (4096, 256), (2048, 8192)]:
    n = G // (h * w)
    x = torch.randint(0, 256, (n, h, w), dtype=torch.uint8, device="cuda")
    sse = torch.empty(n, dtype=torch.float64, device="cuda")
    res = []
    for r in (1, 10, 36):
        ms = t(lambda: A.compress_psnr(x, r, sse=sse))
        res.append(f"r{r}:{G/ms/1e6:.0f}GB/s")
    out = torch.empty((n, h, w), dtype=torch.int16, device="cuda")
    ms = t(lambda: A.forward(x, out=out))
    res.append(f"fwd:{3*G/ms/1e6:.0f}GB/s")
    print(h, w, n, " ".join(res), flush=True)
    del x, out
