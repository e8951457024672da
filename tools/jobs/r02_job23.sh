python -m pytest tests/test_gpu_parity.py -q -m gpu -k "c3_full_size or c4_frames or c5_full_size" --durations=5 2>&1 | tail -12 > gpurun_out/r02_gputests16.txt
