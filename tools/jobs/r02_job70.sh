python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r02_gputests38.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke7.txt 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench13.jsonl 2> gpurun_out/r02_bench13.err
