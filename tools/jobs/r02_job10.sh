python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "quant or determinism or canary or no_writes" 2>&1 | tail -3 > gpurun_out/r02_gputests7.txt
IMAGES=1024 python tools/time_zonal_variants.py default tune_variants/libadct_ringr.so tune_variants/libadct_r3m3.so default > gpurun_out/r02_var_zonal5.txt 2>&1
FRAMES=32 python tools/time_quant_variants.py default tune_variants/libadct_qru.so default tune_variants/libadct_qru.so > gpurun_out/r02_var_quant4.txt 2>&1
