# r02 first GPU call: full GPU test suite (incl. the new multi-rank + step-level tests) + c5 bench.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_r02a.txt 2>&1
tail -5 gpurun_out/gputest_r02a.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cut -c1-3000 gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
python -c "import __graft_entry__ as g; g.smoke()"
