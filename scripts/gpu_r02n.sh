mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 700 python scripts/diag_table2.py hex11x33,hex25x34,grid40,grid60 60,80,100 > gpurun_out/diag_t2.txt 2>&1
cat gpurun_out/diag_t2.txt | tail -60
