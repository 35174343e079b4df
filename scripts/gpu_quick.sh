# quick GPU check: deep-tail parity + config-5 per-step profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "deep_tail or deep_steps or config5 or count_mode or config3" 2>&1 | tail -15
python scripts/prof_step.py c5 3 2>&1 | tee gpurun_out/steps_c5.txt
python scripts/prof_step.py c3-p20 3 2>&1 | head -3
