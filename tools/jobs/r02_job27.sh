python tools/ab_zonal.py --diag --images 32 --rounds 1 default > gpurun_out/r02_diag_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_diag_energy -c 1 -o gpurun_out/r02_prof_diag \
    python tools/ab_zonal.py --diag --images 32 --rounds 1 default > gpurun_out/r02_ncu_diag.log 2>&1
tail -3 gpurun_out/r02_ncu_diag.log
