IMAGES=128 python tools/time_zonal_variants.py default tune_variants/libadct_r1.so default tune_variants/libadct_r1.so > gpurun_out/r02_var_zonal3.txt 2>&1
FRAMES=16 python tools/time_quant_variants.py default tune_variants/libadct_r1.so default tune_variants/libadct_r1.so > gpurun_out/r02_var_quant3.txt 2>&1
