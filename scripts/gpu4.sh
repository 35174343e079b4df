mkdir -p gpurun_out
python scripts/prof_step.py c5 3 > gpurun_out/prof_c5.txt 2>&1
cat gpurun_out/prof_c5.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows|k_step" -s 12 -c 1 -o gpurun_out/prof_c5_v3 python scripts/prof_step.py c5 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
