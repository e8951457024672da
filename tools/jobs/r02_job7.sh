python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/r02_gputests6.txt
IMAGES=128 python tools/time_zonal_variants.py default tune_variants/libadct_r1.so default tune_variants/libadct_r1.so > gpurun_out/r02_var_zonal2.txt 2>&1
FRAMES=16 python tools/time_quant_variants.py default tune_variants/libadct_r1.so > gpurun_out/r02_var_quant2.txt 2>&1
