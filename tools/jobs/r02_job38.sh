python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "compress or determinism or multi" 2>&1 | tail -3 > gpurun_out/r02_gputests23.txt
python tools/ab_zonal.py --images 384 --rounds 5 --rs 22,23,24 default > gpurun_out/r02_ab_r23.txt 2>&1
