# One GPU call: benches of every workload + ncu launch lists + one full capture (config 5).
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep gpurun_out/launches_*.csv gpurun_out/bench_*.json
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --workload c3-p20 --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --workload c2-er-c4 --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1500 python bench.py --workload c4-diamond --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c4d.json 2> gpurun_out/bench_c4d.err
timeout 1500 python bench.py --workload c4-k4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c4k4.json 2> gpurun_out/bench_c4k4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_step.py c5 1 > gpurun_out/prof_c5.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows|k_deep" -s 12 -c 2 -o gpurun_out/prof_c5_full python scripts/prof_step.py c5 1 > gpurun_out/ncu_full.log 2>&1
python scripts/prof_step.py c5 3 > gpurun_out/steps_c5.txt 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_c5.json 2> gpurun_out/bench_ref.err
for f in gpurun_out/bench_*.json; do echo $f; cut -c1-300 $f; done
