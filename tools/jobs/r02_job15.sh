python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r02_gputests12.txt
python tools/time_variants.py > gpurun_out/r02_tv2_default.txt 2>&1
ADCT_LIB=tune_variants/libadct_sw0.so python tools/time_variants.py > gpurun_out/r02_tv2_sw0.txt 2>&1
