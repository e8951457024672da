ADCT_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 3 --images 64 --e2e-images 4 --no-cpu-baseline > gpurun_out/r02_bench_2rank_functional.jsonl 2> gpurun_out/r02_bench_2rank_functional.err
echo "rc=$?" >> gpurun_out/r02_bench_2rank_functional.err
