python tools/ab_zonal.py --images 384 --rounds 7 --rs 19,20,21,22,23 default tune_variants/libadct_res19.so > gpurun_out/r02_ab_res19.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 19,20,21,22,23 tune_variants/libadct_res19.so default >> gpurun_out/r02_ab_res19.txt 2>&1
