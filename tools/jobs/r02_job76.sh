python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "compress or determinism or multi or extremes or ragged" 2>&1 | tail -3 > gpurun_out/r02_gputests41.txt
python tools/ab_zonal.py --images 384 --rounds 7 --rs 23,26,28,30,36,40,45,50 default tune_variants/libadct_nopc.so > gpurun_out/r02_ab_pc.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 23,26,28,30,36,40,45,50 tune_variants/libadct_nopc.so default >> gpurun_out/r02_ab_pc.txt 2>&1
