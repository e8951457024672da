python tools/ab_zonal.py --images 512 --rounds 9 default tune_variants/libadct_h3.so tune_variants/libadct_s1.so > gpurun_out/r02_ab_h3s1.txt 2>&1
python tools/ab_zonal.py --images 512 --rounds 9 tune_variants/libadct_s1.so tune_variants/libadct_h3.so default >> gpurun_out/r02_ab_h3s1.txt 2>&1
