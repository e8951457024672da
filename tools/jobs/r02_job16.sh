IMAGES=1024 python tools/time_zonal_variants.py default tune_variants/libadct_h3.so default tune_variants/libadct_h3.so > gpurun_out/r02_var_zonal9.txt 2>&1
