python tools/ab_zonal.py --images 512 --rounds 7 default tune_variants/libadct_st3.so tune_variants/libadct_ds3.so > gpurun_out/r02_ab_st3ds3.txt 2>&1
python tools/ab_zonal.py --images 512 --rounds 7 tune_variants/libadct_ds3.so tune_variants/libadct_st3.so default >> gpurun_out/r02_ab_st3ds3.txt 2>&1
