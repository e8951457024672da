python tools/ab_zonal.py --images 384 --rounds 7 --rs 2,3,6,10,12,15,18,21,22 default tune_variants/libadct_sm4.so > gpurun_out/r02_ab_sm4.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 2,3,6,10,12,15,18,21,22 tune_variants/libadct_sm4.so default >> gpurun_out/r02_ab_sm4.txt 2>&1
