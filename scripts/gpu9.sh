mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_step.py c5 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4d.csv python scripts/prof_step.py c4-diamond 1 > /dev/null 2>&1
python scripts/ncu_traffic.py gpurun_out/launches_c5.csv c5 | head -3
python scripts/ncu_traffic.py gpurun_out/launches_c4d.csv c4-diamond | head -3
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 1200 python bench.py --workload c4-diamond --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c4d.json 2> gpurun_out/bench_c4d.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c5.json 2> gpurun_out/bench_ref_c5.err
tail -2 gpurun_out/bench_c5.err gpurun_out/bench_c4d.err gpurun_out/bench_ref_c5.err
cat gpurun_out/bench_c5.json gpurun_out/bench_c4d.json gpurun_out/bench_ref_c5.json
