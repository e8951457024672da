ADCT_LIB=tune_variants/libadct_rs1.so python tools/time_variants.py > gpurun_out/r02_tv8_rs1.txt 2>&1
ADCT_LIB=tune_variants/libadct_rs3.so python tools/time_variants.py > gpurun_out/r02_tv8_rs3.txt 2>&1
python -m pytest tests/test_gpu_parity.py -q -m gpu -k "recon" 2>&1 | tail -2 > gpurun_out/r02_gputests35.txt
