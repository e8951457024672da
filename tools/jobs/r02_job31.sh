python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench7.jsonl 2> gpurun_out/r02_bench7.err
