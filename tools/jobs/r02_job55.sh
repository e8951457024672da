python tools/time_variants.py > gpurun_out/r02_tv5_default.txt 2>&1
ADCT_LIB=tune_variants/libadct_s1.so python tools/time_variants.py > gpurun_out/r02_tv5_s1.txt 2>&1
ADCT_LIB=tune_variants/libadct_h3.so python tools/time_variants.py > gpurun_out/r02_tv5_h3.txt 2>&1
