python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r02_gputests9.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench4.jsonl 2> gpurun_out/r02_bench4.err
tail -2 gpurun_out/r02_bench4.err
