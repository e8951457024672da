python tools/ab_zonal.py --images 384 --rounds 7 --rs 28,30,36,40 default tune_variants/libadct_p2.so > gpurun_out/r02_ab_p2.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 28,30,36,40 tune_variants/libadct_p2.so default >> gpurun_out/r02_ab_p2.txt 2>&1
