python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "compress or determinism or multi or extremes or ragged" 2>&1 | tail -3 > gpurun_out/r02_gputests43.txt
python tools/ab_zonal.py --images 384 --rounds 7 --rs 24,26,27,28,30,32,35,36 default tune_variants/libadct_nop2.so > gpurun_out/r02_ab_p2c.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 24,26,27,28,30,32,35,36 tune_variants/libadct_nop2.so default >> gpurun_out/r02_ab_p2c.txt 2>&1
