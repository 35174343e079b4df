mkdir -p gpurun_out
python scripts/prof_step.py c5 3 2>&1 | grep -E "config5|step 1[0-3]" | cut -c1-150
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python -c "import json; d=json.load(open('gpurun_out/bench_c5.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
python scripts/prof_step.py c5 3 2>&1 | grep -E "config5|step 1[0-3]" | cut -c1-150
