python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py tests/test_dist_gpu.py -q -m gpu -x -k "multi or host or determinism" 2>&1 | tail -3 > gpurun_out/r02_gputests14.txt
IMAGES=256 python tools/time_multi_variants.py default tune_variants/libadct_nopair.so default tune_variants/libadct_nopair.so > gpurun_out/r02_var_multi1.txt 2>&1
