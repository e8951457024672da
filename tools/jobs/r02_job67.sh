python tools/ab_zonal.py --images 768 --rounds 9 --rs 1 default tune_variants/libadct_a34.so tune_variants/libadct_a43.so tune_variants/libadct_a35.so > gpurun_out/r02_ab_r1ring.txt 2>&1
python tools/ab_zonal.py --images 768 --rounds 9 --rs 1 tune_variants/libadct_a35.so tune_variants/libadct_a43.so tune_variants/libadct_a34.so default >> gpurun_out/r02_ab_r1ring.txt 2>&1
