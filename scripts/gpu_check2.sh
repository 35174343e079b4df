mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python scripts/diag_e2e.py > gpurun_out/diag_e2e.txt 2>&1; cat gpurun_out/diag_e2e.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_pool.txt 2>&1
tail -3 gpurun_out/gputest_pool.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5_pool.json 2> gpurun_out/bench_c5_pool.err
python -c "import json; d=json.loads(open('gpurun_out/bench_c5_pool.json').read()); print(d['value'], d['ms_per_step'], d['e2e'])"
