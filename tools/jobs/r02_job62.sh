python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "recon or u8 or no_writes or canary" 2>&1 | tail -3 > gpurun_out/r02_gputests34.txt
python tools/time_variants.py > gpurun_out/r02_tv6_default.txt 2>&1
