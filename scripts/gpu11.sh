timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
DM_BENCH_DEVICE=0 DM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --workload c4-diamond-s18 --gpus 2 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/bench_2rank_c4.json 2> gpurun_out/bench_2rank_c4.err
tail -3 gpurun_out/bench_2rank_c4.err; head -c 900 gpurun_out/bench_2rank_c4.json
