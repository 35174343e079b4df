mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for w in c5 c3-p20 c2-er-c4 c4-k4-s16 c4-diamond-s18; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2> gpurun_out/bc_$w.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['roofline']['kernel'])" || tail -3 gpurun_out/bc_$w.err
done
