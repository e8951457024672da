python -m pytest tests/test_gpu_parity.py -q -m gpu -k "extremes" 2>&1 | tail -3 > gpurun_out/r02_gputests33.txt
