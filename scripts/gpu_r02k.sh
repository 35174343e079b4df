# key-grouped count kernel: parity + per-step times + bench + full capture
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_motifs.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "motif or config5 or heavy_hex or config3" > gpurun_out/gputest_grp.txt 2>&1
tail -3 gpurun_out/gputest_grp.txt
python scripts/prof_step.py c5 3 > gpurun_out/steps_c5.txt 2>&1
cat gpurun_out/steps_c5.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cut -c1-300 gpurun_out/bench_c5.json; tail -n 2 gpurun_out/bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_step.py c5 1 > gpurun_out/prof_c5.txt 2>&1
python scripts/ncu_traffic.py gpurun_out/launches_c5.csv c5x | head -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_table_grouped" -c 1 -o gpurun_out/prof_c5_grp python scripts/prof_step.py c5 1 > gpurun_out/ncu_grp.log 2>&1
tail -1 gpurun_out/ncu_grp.log
