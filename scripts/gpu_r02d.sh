# r02 measurement call: GPU parity suite, config-5 bench, launch list + full capture of the top kernels.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --ignore tests/test_gpu_table2.py -p no:cacheprovider --durations=15 > gpurun_out/gputest.txt 2>&1
tail -5 gpurun_out/gputest.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cut -c1-1500 gpurun_out/bench_c5.json; tail -n 3 gpurun_out/bench_c5.err
python scripts/prof_step.py c5 3 > gpurun_out/steps_c5.txt 2>&1
cat gpurun_out/steps_c5.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_step.py c5 1 > gpurun_out/prof_c5.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_table|k_rows" -c 4 -o gpurun_out/prof_c5_full python scripts/prof_step.py c5 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
