python tools/ab_zonal.py --images 384 --rounds 7 --rs 29,32,36,40,45,50 default tune_variants/libadct_r4a.so tune_variants/libadct_r4b.so > gpurun_out/r02_ab_rsm4.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 29,32,36,40,45,50 tune_variants/libadct_r4b.so tune_variants/libadct_r4a.so default >> gpurun_out/r02_ab_rsm4.txt 2>&1
