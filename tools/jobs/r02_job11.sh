python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/r02_gputests8.txt
python tools/time_variants.py > gpurun_out/r02_tv_default.txt 2>&1
ADCT_LIB=tune_variants/libadct_ringu.so python tools/time_variants.py > gpurun_out/r02_tv_ringu.txt 2>&1
IMAGES=1024 python tools/time_zonal_variants.py default tune_variants/libadct_r3m3.so default tune_variants/libadct_r3m3.so > gpurun_out/r02_var_zonal6.txt 2>&1
FRAMES=32 python tools/time_quant_variants.py default tune_variants/libadct_q4.so default tune_variants/libadct_q4.so > gpurun_out/r02_var_quant5.txt 2>&1
