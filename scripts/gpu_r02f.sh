# vertex-mask count kernel: parity (table steps) + config-5 bench + per-step times.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_motifs.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "motif or config5 or heavy_hex or config3" > gpurun_out/gputest_vm.txt 2>&1
tail -5 gpurun_out/gputest_vm.txt
python scripts/prof_step.py c5 3 > gpurun_out/steps_c5.txt 2>&1
cat gpurun_out/steps_c5.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cut -c1-400 gpurun_out/bench_c5.json; tail -n 3 gpurun_out/bench_c5.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_table_vm" -c 1 -o gpurun_out/prof_c5_vm python scripts/prof_step.py c5 1 > gpurun_out/ncu_vm.log 2>&1
tail -2 gpurun_out/ncu_vm.log
