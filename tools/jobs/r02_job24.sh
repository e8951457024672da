python -m pytest tests/test_gpu_parity.py -q -m gpu -k "c5_full_size" --durations=3 2>&1 | tail -8 > gpurun_out/r02_gputests17.txt
