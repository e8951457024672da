python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "sse576 or exact or no_writes" 2>&1 | tail -3 > gpurun_out/r02_gputests39.txt
python tools/time_variants.py > gpurun_out/r02_tv9_default.txt 2>&1
