python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "sse576 or exact" 2>&1 | tail -3 > gpurun_out/r02_gputests18.txt
python tools/time_variants.py > gpurun_out/r02_tv3_default.txt 2>&1
ADCT_LIB=tune_variants/libadct_exold.so python tools/time_variants.py > gpurun_out/r02_tv3_exold.txt 2>&1
