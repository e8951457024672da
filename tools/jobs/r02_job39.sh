python tools/ab_zonal.py --images 384 --rounds 7 --rs 2,3,4,5,6,7,8,9,10,11 default tune_variants/libadct_h3.so tune_variants/libadct_s0.so > gpurun_out/r02_ab_lowr.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 2,3,4,5,6,7,8,9,10,11 tune_variants/libadct_s0.so tune_variants/libadct_h3.so default >> gpurun_out/r02_ab_lowr.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 5 --rs 24,26,28,30,32,36,40,45 default tune_variants/libadct_s0.so > gpurun_out/r02_ab_highr.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 5 --rs 24,26,28,30,32,36,40,45 tune_variants/libadct_s0.so default >> gpurun_out/r02_ab_highr.txt 2>&1
