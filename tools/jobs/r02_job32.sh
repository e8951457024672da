python -m pytest tests/test_gpu_parity.py -q -m gpu -k "diag or sweep or extreme" 2>&1 | tail -3 > gpurun_out/r02_gputests20.txt
python - > gpurun_out/r02_diag_prefix_timing.txt 2>&1 <<'PY'
import sys, json, torch
sys.path.insert(0, '.')
import paper_1402_6034_b200 as A
from synth import images as S
peak = json.load(open('MEASURED_PEAKS.json'))['hbm_gbs']
x = S.device_mixed(256, 4096, 4096, device='cuda')
en = torch.empty((256, 16), dtype=torch.int64, device='cuda')
for rm in (64, 36, 64, 36):
    A.diag_energy(x, energy=en, r_max=rm); torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): A.diag_energy(x, energy=en, r_max=rm)
        e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / 3)
    print(f"diag energy r_max={rm}: {best:.3f} ms  HBM frac {x.numel() / (best * 1e-3) / 1e9 / peak:.4f}")
PY
