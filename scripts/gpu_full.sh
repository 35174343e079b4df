mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python scripts/prof_step.py c5 3 2>&1 | tee gpurun_out/steps_c5.txt | cut -c1-150
