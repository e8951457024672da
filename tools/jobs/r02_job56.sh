python tools/ab_zonal.py --images 384 --rounds 7 --rs 3,5,6,8,9,10 default tune_variants/libadct_grp.so > gpurun_out/r02_ab_grp.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 3,5,6,8,9,10 tune_variants/libadct_grp.so default >> gpurun_out/r02_ab_grp.txt 2>&1
