python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r02_gputests40.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke8.txt 2>&1
