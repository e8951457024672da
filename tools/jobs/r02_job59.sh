python - > gpurun_out/r02_h2d_raw.txt 2>&1 <<'PY'
import torch
h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
d = torch.empty(1 << 30, dtype=torch.uint8, device='cuda')
for chunk in (1 << 30, 128 << 20, 32 << 20):
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for o in range(0, 1 << 30, chunk):
            d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
        e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"H2D pinned 1 GiB in {chunk >> 20} MiB chunks: {best:.2f} ms = {(1 << 30) / (best * 1e-3) / 1e9:.1f} GB/s")
PY
