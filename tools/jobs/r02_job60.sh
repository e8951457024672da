python -m pytest tests/test_gpu_parity.py -q -m gpu -k "ragged" --durations=3 2>&1 | tail -6 > gpurun_out/r02_gputests32.txt
