mkdir -p gpurun_out
for wl in c4-diamond-s16 c4-k4-s16 c4-diamond-s18 c3-p20 c2-er-c4; do
  timeout 300 python scripts/prof_step.py $wl 2 2>&1 | tail -8
done
timeout 600 python scripts/prof_step.py c4-diamond 1 2>&1 | tail -5
