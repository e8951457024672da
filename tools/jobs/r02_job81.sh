python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r02_gputests44.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke10.txt 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench15.jsonl 2> gpurun_out/r02_bench15.err
python tools/prof_compress.py --n 32 --r 28 --reps 1 > gpurun_out/r02_prof_plain8.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_compress -c 1 -o gpurun_out/r02_prof_compress8 \
    python tools/prof_compress.py --n 32 --r 28 --reps 1 > gpurun_out/r02_ncu_full8.log 2>&1
