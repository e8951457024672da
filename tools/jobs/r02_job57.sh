python tools/ab_zonal.py --images 768 --rounds 9 --rs 1 default tune_variants/libadct_f8.so tune_variants/libadct_f4.so > gpurun_out/r02_ab_f16r1.txt 2>&1
python tools/ab_zonal.py --images 768 --rounds 9 --rs 1 tune_variants/libadct_f4.so tune_variants/libadct_f8.so default >> gpurun_out/r02_ab_f16r1.txt 2>&1
