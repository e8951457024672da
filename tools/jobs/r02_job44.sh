python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r02_gputests27.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke3.txt 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench9.jsonl 2> gpurun_out/r02_bench9.err
python tools/prof_compress.py --n 32 --r 3,15 --reps 1 > gpurun_out/r02_prof_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_compress -c 2 -o gpurun_out/r02_prof_compress3 \
    python tools/prof_compress.py --n 32 --r 3,15 --reps 1 > gpurun_out/r02_ncu_full3.log 2>&1
