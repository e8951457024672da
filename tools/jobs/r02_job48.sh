python tools/ab_zonal.py --images 384 --rounds 7 --rs 18,19,20,21,22 default tune_variants/libadct_a3.so tune_variants/libadct_a4.so tune_variants/libadct_a5.so > gpurun_out/r02_ab_sm4b.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 18,19,20,21,22 tune_variants/libadct_a5.so tune_variants/libadct_a4.so tune_variants/libadct_a3.so default >> gpurun_out/r02_ab_sm4b.txt 2>&1
