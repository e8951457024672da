python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "compress or determinism or multi" 2>&1 | tail -3 > gpurun_out/r02_gputests22.txt
python tools/ab_zonal.py --images 512 --rounds 9 default tune_variants/libadct_prev.so > gpurun_out/r02_ab_hyb.txt 2>&1
python tools/ab_zonal.py --images 512 --rounds 9 tune_variants/libadct_prev.so default >> gpurun_out/r02_ab_hyb.txt 2>&1
