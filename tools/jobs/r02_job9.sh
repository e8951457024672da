IMAGES=1024 python tools/time_zonal_variants.py default tune_variants/libadct_r1.so > gpurun_out/r02_var_zonal4.txt 2>&1
python tools/prof_compress.py --n 32 --r 1,3,6,10,15,21,28,36 --reps 1 --quant > gpurun_out/r02_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_compress -c 9 -o gpurun_out/r02_prof_compress \
    python tools/prof_compress.py --n 32 --r 1,3,6,10,15,21,28,36 --reps 1 --quant > gpurun_out/r02_ncu_full.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_bench_ncuplain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ncu_launches.log 2>&1
echo done
