python tools/traffic_ceiling.py > gpurun_out/r02_c3_traffic_ceiling.txt 2>&1
