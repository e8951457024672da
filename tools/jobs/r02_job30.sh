python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "sse576 or exact" 2>&1 | tail -3 > gpurun_out/r02_gputests19.txt
