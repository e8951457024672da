./tools/microbench/readbw > gpurun_out/r02_readbw.txt 2>&1
