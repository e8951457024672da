python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -m gpu -k "compress or determinism or multi" 2>&1 | tail -3 > gpurun_out/r02_gputests30.txt
python tools/prof_compress.py --n 32 --r 15 --reps 1 > gpurun_out/r02_prof_plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_compress -c 1 -o gpurun_out/r02_prof_compress5 \
    python tools/prof_compress.py --n 32 --r 15 --reps 1 > gpurun_out/r02_ncu_full5.log 2>&1
