mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cut -c1-4000 gpurun_out/bench_c5.json; tail -n 3 gpurun_out/bench_c5.err
