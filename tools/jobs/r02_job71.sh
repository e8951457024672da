python tools/prof_compress.py --n 32 --r 6,10 --reps 1 > gpurun_out/r02_prof_plain6.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_compress -c 2 -o gpurun_out/r02_prof_compress6 \
    python tools/prof_compress.py --n 32 --r 6,10 --reps 1 > gpurun_out/r02_ncu_full6.log 2>&1
