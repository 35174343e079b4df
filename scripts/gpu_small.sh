mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2 3; do timeout 300 python bench.py --workload c3-p20 --steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['ms_per_step'])"; done
python scripts/prof_step.py c3-p20 5 2>&1 | tail -12
python scripts/prof_step.py c2-er-c4 5 2>&1 | tail -8
