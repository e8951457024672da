python tools/ab_zonal.py --images 384 --rounds 7 --rs 11,12,13,14,15,16,17,18,19,20,21,22,23 default tune_variants/libadct_h3.so > gpurun_out/r02_ab_h3_mid.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 11,12,13,14,15,16,17,18,19,20,21,22,23 tune_variants/libadct_h3.so default >> gpurun_out/r02_ab_h3_mid.txt 2>&1
