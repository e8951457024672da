python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r02_gputests31.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke5.txt 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench11.jsonl 2> gpurun_out/r02_bench11.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_bench_ncuplain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv --log-file gpurun_out/r02_launches3.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ncu_launches3.log 2>&1
