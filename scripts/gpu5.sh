mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_step.py c5 1 > /dev/null 2>&1
python scripts/ncu_traffic.py gpurun_out/launches_c5.csv c5
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -2 gpurun_out/bench_c5.err; cat gpurun_out/bench_c5.json
