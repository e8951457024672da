./tools/microbench/mix12 > gpurun_out/r02_mix12.txt 2>&1
