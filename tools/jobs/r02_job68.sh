python -m pytest tests/test_gpu_parity.py -q -m gpu -k "compress_every_r or ragged or c5_full or determinism" 2>&1 | tail -3 > gpurun_out/r02_gputests37.txt
