python tools/time_variants.py > gpurun_out/r02_tv4_default.txt 2>&1
ADCT_LIB=tune_variants/libadct_exs.so python tools/time_variants.py > gpurun_out/r02_tv4_exs.txt 2>&1
python tools/time_variants.py > gpurun_out/r02_tv4_default2.txt 2>&1
