# quick cycle: table-step parity suites + config-5 per-step times + bench
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_motifs.py tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_table2.py -x -q -p no:cacheprovider > gpurun_out/gputest_check.txt 2>&1
tail -3 gpurun_out/gputest_check.txt
python scripts/prof_step.py c5 3 > gpurun_out/steps_c5.txt 2>&1; tail -2 gpurun_out/steps_c5.txt
timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c5_check.json 2> gpurun_out/bench_c5_check.err
cut -c1-260 gpurun_out/bench_c5_check.json
