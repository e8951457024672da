python tools/ab_zonal.py --images 384 --rounds 7 --rs 15,18,21 default tune_variants/libadct_nomirb.so > gpurun_out/r02_ab_nomirb.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 15,18,21 tune_variants/libadct_nomirb.so default >> gpurun_out/r02_ab_nomirb.txt 2>&1
