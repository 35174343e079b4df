mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_apex.py -x -q -p no:cacheprovider > gpurun_out/gputest_apex.txt 2>&1
tail -2 gpurun_out/gputest_apex.txt
timeout 900 python -m pytest tests/test_gpu_table2.py -q -p no:cacheprovider --durations=0 -x -k "hex11x33" > gpurun_out/gputest_t2a.txt 2>&1
tail -25 gpurun_out/gputest_t2a.txt
timeout 600 python bench.py --workload c4-diamond --motifs apex --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c4d_apex.json 2> gpurun_out/bench_c4d_apex.err
cut -c1-300 gpurun_out/bench_c4d_apex.json; tail -2 gpurun_out/bench_c4d_apex.err
