IMAGES=256 python tools/time_multi_variants.py default tune_variants/libadct_u2.so tune_variants/libadct_nosplit.so default tune_variants/libadct_u2.so > gpurun_out/r02_var_multi3.txt 2>&1
