python __graft_entry__.py smoke
DM_BENCH_DEVICE=0 DM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | cut -c1-400
DM_BENCH_DEVICE=0 DM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 2 --warmup 3 --workload c4-diamond-s18 --no-cpu-baseline 2>&1 | grep '^{' | cut -c1-600
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 2>&1 | grep '^{' | cut -c1-300
