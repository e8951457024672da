python -m pytest tests/test_gpu_parity.py -q -m gpu -k "multi" 2>&1 | tail -3 > gpurun_out/r02_gputests25.txt
IMAGES=256 python tools/time_multi_variants.py default tune_variants/libadct_sp2.so tune_variants/libadct_sp4.so tune_variants/libadct_nosplit.so default > gpurun_out/r02_var_multi2.txt 2>&1
