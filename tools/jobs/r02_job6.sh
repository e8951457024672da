./tools/microbench/regbank > gpurun_out/r02_regbank2.txt 2>&1
python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/r02_gputests5.txt
IMAGES=128 python tools/time_zonal_variants.py default tune_variants/libadct_nomirb.so tune_variants/libadct_resid21.so > gpurun_out/r02_var_zonal1.txt 2>&1
FRAMES=16 python tools/time_quant_variants.py default tune_variants/libadct_qlo.so tune_variants/libadct_nomirb.so > gpurun_out/r02_var_quant1.txt 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench3.jsonl 2> gpurun_out/r02_bench3.err
tail -2 gpurun_out/r02_bench3.err
