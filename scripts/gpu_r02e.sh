# apex table (a1b) parity + K4 bench, k_table full capture on config 5.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_apex.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/gputest_apex.txt 2>&1
tail -15 gpurun_out/gputest_apex.txt
timeout 900 python bench.py --workload c4-k4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c4k4.json 2> gpurun_out/bench_c4k4.err
cut -c1-600 gpurun_out/bench_c4k4.json; tail -n 3 gpurun_out/bench_c4k4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_step.py c5 1 > gpurun_out/prof_c5.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_table" -c 4 -o gpurun_out/prof_c5_table python scripts/prof_step.py c5 1 > gpurun_out/ncu_table.log 2>&1
tail -2 gpurun_out/ncu_table.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pairs_apex|k_apex" -c 3 -o gpurun_out/prof_k4s16 python scripts/prof_step.py c4-k4-s16 1 > gpurun_out/ncu_k4.log 2>&1
tail -3 gpurun_out/ncu_k4.log
