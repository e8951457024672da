python tools/ab_zonal.py --images 768 --rounds 9 --rs 2,3 default tune_variants/libadct_b42.so tune_variants/libadct_b43.so tune_variants/libadct_b22.so > gpurun_out/r02_ab_r3ring.txt 2>&1
python tools/ab_zonal.py --images 768 --rounds 9 --rs 2,3 tune_variants/libadct_b22.so tune_variants/libadct_b43.so tune_variants/libadct_b42.so default >> gpurun_out/r02_ab_r3ring.txt 2>&1
