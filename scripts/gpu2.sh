mkdir -p gpurun_out
python scripts/prof_step.py c5 3 > gpurun_out/prof_c5.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_step.py c5 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 27 -c 1 -o gpurun_out/prof_c5_write13 python scripts/prof_step.py c5 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
cat gpurun_out/prof_c5.txt
timeout 900 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
tail -15 gpurun_out/pytest_gpu.txt
