timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/diag_small.py 2>&1 | tail -4
python scripts/prof_step.py c5 3 | head -1
