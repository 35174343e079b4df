mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tail" -c 1 -o gpurun_out/prof_tail python scripts/prof_step.py c5 1 > gpurun_out/ncu_tail.log 2>&1
tail -3 gpurun_out/ncu_tail.log
