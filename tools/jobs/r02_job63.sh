python tools/time_variants.py > gpurun_out/r02_tv7_default.txt 2>&1
ADCT_LIB=tune_variants/libadct_rs1.so python tools/time_variants.py > gpurun_out/r02_tv7_rs1.txt 2>&1
