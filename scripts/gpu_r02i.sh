# table-step flush change: parity + per-step times + bench
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_motifs.py tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -p no:cacheprovider > gpurun_out/gputest_flush.txt 2>&1
tail -3 gpurun_out/gputest_flush.txt
python scripts/prof_step.py c5 3 > gpurun_out/steps_c5.txt 2>&1
cat gpurun_out/steps_c5.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cut -c1-300 gpurun_out/bench_c5.json; tail -n 3 gpurun_out/bench_c5.err
