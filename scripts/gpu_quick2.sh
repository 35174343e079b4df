mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "deep_tail or deep_steps or config5 or count_mode or config3" 2>&1 | tail -5
python scripts/prof_step.py c5 3 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tail" -c 1 -o gpurun_out/prof_tail python scripts/prof_step.py c5 1 > gpurun_out/ncu_tail.log 2>&1
