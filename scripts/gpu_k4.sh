mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_apex.py -x -q -p no:cacheprovider > gpurun_out/gputest_apex.txt 2>&1
tail -2 gpurun_out/gputest_apex.txt
python scripts/prof_step.py c4-k4-s16 3 > gpurun_out/steps_c4k4s16.txt 2>&1; tail -1 gpurun_out/steps_c4k4s16.txt
timeout 900 python bench.py --workload c4-k4 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c4k4_t.json 2> gpurun_out/bench_c4k4_t.err
cut -c1-260 gpurun_out/bench_c4k4_t.json
