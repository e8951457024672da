python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "compress or determinism or multi" 2>&1 | tail -3 > gpurun_out/r02_gputests24.txt
python tools/ab_zonal.py --images 384 --rounds 5 --rs 2,3,4,7,8 default tune_variants/libadct_s0.so > gpurun_out/r02_ab_lowr2.txt 2>&1
