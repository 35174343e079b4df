mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --workload c3-p20 --steps 50 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
rm -f gpurun_out/launches_c5.csv gpurun_out/prof_c5_full.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_step.py c5 1 > gpurun_out/prof_c5.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows|k_deep" -s 12 -c 2 -o gpurun_out/prof_c5_full python scripts/prof_step.py c5 1 > gpurun_out/ncu_full.log 2>&1
python scripts/prof_step.py c5 3 > gpurun_out/steps_c5.txt 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench_c5.json')); print(d['value'], d['ms_per_step'], d['roofline']['by_kind'])"
