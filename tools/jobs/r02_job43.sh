python -m pytest tests/test_gpu_parity.py -q -m gpu -k "multi or host" 2>&1 | tail -3 > gpurun_out/r02_gputests26.txt
IMAGES=256 python tools/time_multi_variants.py default tune_variants/libadct_u2.so tune_variants/libadct_nosplit.so default tune_variants/libadct_u2.so > gpurun_out/r02_var_multi3.txt 2>&1
