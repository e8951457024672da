FRAMES=32 python tools/time_quant_variants.py default tune_variants/libadct_q3.so default tune_variants/libadct_q3.so > gpurun_out/r02_var_quant8.txt 2>&1
