set -x
DM_BENCH_DEVICE=0 DM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
tail -5 gpurun_out/bench_2rank.err; cat gpurun_out/bench_2rank.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_ref_2rank.json 2> gpurun_out/bench_ref_2rank.err
tail -3 gpurun_out/bench_ref_2rank.err; cat gpurun_out/bench_ref_2rank.json
