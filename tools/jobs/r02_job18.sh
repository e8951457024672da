python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r02_gputests13.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench5.jsonl 2> gpurun_out/r02_bench5.err
python tools/ab_zonal.py --images 512 --quant-frames 32 default > gpurun_out/r02_ab_default.txt 2>&1
python tools/prof_compress.py --n 32 --r 1,3,6,10,15,21,28,36 --reps 1 --quant > gpurun_out/r02_prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_compress -c 9 -o gpurun_out/r02_prof_compress2 \
    python tools/prof_compress.py --n 32 --r 1,3,6,10,15,21,28,36 --reps 1 --quant > gpurun_out/r02_ncu_full2.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_bench_ncuplain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv --log-file gpurun_out/r02_launches2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ncu_launches2.log 2>&1
echo done
