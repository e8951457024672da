python tools/ab_zonal.py --images 384 --rounds 7 --rs 24,27,28,29,30,33,36 default tune_variants/libadct_p2a.so tune_variants/libadct_p2b.so > gpurun_out/r02_ab_p2b.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 24,27,28,29,30,33,36 tune_variants/libadct_p2b.so tune_variants/libadct_p2a.so default >> gpurun_out/r02_ab_p2b.txt 2>&1
