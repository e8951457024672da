python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -x -k "compress or quant or determinism or multi" 2>&1 | tail -3 > gpurun_out/r02_gputests11.txt
IMAGES=1024 python tools/time_zonal_variants.py default tune_variants/libadct_ng1.so tune_variants/libadct_ng2.so tune_variants/libadct_s0.so default tune_variants/libadct_ng1.so > gpurun_out/r02_var_zonal8.txt 2>&1
FRAMES=32 python tools/time_quant_variants.py default tune_variants/libadct_s0.so > gpurun_out/r02_var_quant7.txt 2>&1
