python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py tests/test_dist_gpu.py -q -m gpu -k "compress or determinism or multi or dist" 2>&1 | tail -3 > gpurun_out/r02_gputests28.txt
python tools/ab_zonal.py --images 512 --rounds 7 default > gpurun_out/r02_ab_final1.txt 2>&1
