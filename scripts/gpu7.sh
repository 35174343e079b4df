mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for wl in c4-diamond-s16 c4-k4-s16 c4-diamond-s18; do
  timeout 300 python scripts/prof_step.py $wl 2 2>&1 | head -4
done
timeout 600 python scripts/prof_step.py c4-diamond 2 2>&1 | tail -4
timeout 600 python scripts/prof_step.py c4-k4 2 2>&1 | tail -4
