# r02 evidence run: GPU parity suite, smoke, every bench workload, the reference arm, ncu launch
# lists and full captures of the dominant kernels (config 5: k_table; config 4: k_pairs_apex).
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep gpurun_out/launches_*.csv gpurun_out/bench_*.json gpurun_out/steps_*.txt
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/gputest.txt 2>&1
tail -4 gpurun_out/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --workload c3-p20 --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --workload c2-er-c4 --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1500 python bench.py --workload c4-diamond --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c4d.json 2> gpurun_out/bench_c4d.err
timeout 1500 python bench.py --workload c4-k4 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c4k4.json 2> gpurun_out/bench_c4k4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_c5.json 2> gpurun_out/bench_ref.err
for f in gpurun_out/bench_*.json; do echo $f; cut -c1-260 $f; done
python scripts/prof_step.py c5 3 > gpurun_out/steps_c5.txt 2>&1
python scripts/prof_step.py c4-k4-s16 2 > gpurun_out/steps_c4k4s16.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_step.py c5 1 > gpurun_out/prof_c5.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4-k4.csv python scripts/prof_step.py c4-k4 1 > gpurun_out/prof_c4k4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4-diamond.csv python scripts/prof_step.py c4-diamond 1 > gpurun_out/prof_c4d.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_table" -c 4 -o gpurun_out/prof_c5_full python scripts/prof_step.py c5 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pairs_apex" -c 1 -o gpurun_out/prof_c4k4s16_full python scripts/prof_step.py c4-k4-s16 1 > gpurun_out/ncu_k4.log 2>&1
tail -1 gpurun_out/ncu_full.log gpurun_out/ncu_k4.log
# multi-rank bench path on one device (gloo collectives; the data path is the library's)
DM_BENCH_DEVICE=0 DM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/multi_c5.txt 2>&1
DM_BENCH_DEVICE=0 DM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 2 --warmup 3 --workload c4-diamond-s18 --no-cpu-baseline > gpurun_out/multi_c4d.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/multi_ref.txt 2>&1
grep -h '^{' gpurun_out/multi_*.txt | cut -c1-300
