# every bench workload + the reference arm on the current build (bench lines for profiles/)
mkdir -p gpurun_out
rm -f gpurun_out/bench_*.json
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --workload c3-p20 --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --workload c2-er-c4 --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1500 python bench.py --workload c4-diamond --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c4d.json 2> gpurun_out/bench_c4d.err
timeout 1500 python bench.py --workload c4-k4 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c4k4.json 2> gpurun_out/bench_c4k4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_c5.json 2> gpurun_out/bench_ref.err
for f in gpurun_out/bench_*.json; do echo $f; cut -c1-200 $f; done
