python tools/ab_zonal.py --images 384 --rounds 7 --rs 23,25,27,28 default tune_variants/libadct_nohc.so > gpurun_out/r02_ab_nohc.txt 2>&1
python tools/ab_zonal.py --images 384 --rounds 7 --rs 23,25,27,28 tune_variants/libadct_nohc.so default >> gpurun_out/r02_ab_nohc.txt 2>&1
