python tools/ab_zonal.py --images 384 --rounds 7 --rs 14,15,16,17 default tune_variants/libadct_s14.so > gpurun_out/r02_ab_s14.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 14,15,16,17 tune_variants/libadct_s14.so default >> gpurun_out/r02_ab_s14.txt 2>&1
