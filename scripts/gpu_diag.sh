mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python scripts/diag_e2e.py > gpurun_out/diag_e2e.txt 2>&1; cat gpurun_out/diag_e2e.txt
