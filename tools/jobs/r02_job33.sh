python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r02_gputests21.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke2.txt 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench8.jsonl 2> gpurun_out/r02_bench8.err
python tools/ab_zonal.py --diag --images 32 --rounds 1 default > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_diag_energy|k_compress_sweep_inc|k_compress_exact" -c 3 -o gpurun_out/r02_prof_secondary \
    python - > gpurun_out/r02_ncu_secondary.log 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1402_6034_b200 as A
from synth import images as S
x = S.device_mixed(32, 4096, 4096, device='cuda')
A.diag_energy(x, r_max=36)
A.compress_psnr_multi(x, (1, 3, 6, 10, 15, 21, 28, 36))
A.compress_sse576(x, 10)
torch.cuda.synchronize()
print("ok")
PY
tail -2 gpurun_out/r02_ncu_secondary.log
