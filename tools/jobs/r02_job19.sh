python tools/ab_zonal.py --images 512 --rounds 9 default tune_variants/libadct_m3.so > gpurun_out/r02_ab_m3.txt 2>&1
python tools/ab_zonal.py --images 512 --rounds 9 tune_variants/libadct_m3.so default > gpurun_out/r02_ab_m3b.txt 2>&1
