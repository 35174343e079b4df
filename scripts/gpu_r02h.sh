# motif-set sweep on config 5 (device ms per dm_match, per-step kernel ms)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
rm -f gpurun_out/motif_sweep.txt
for m in M2,M7 M2,M8 M2,M3,M8 M2,M6 M2,M3,M7 M2,M5 M2,M4 M2,M3,M6 M2,M12-O,M7; do
  timeout 120 python scripts/motif_bench.py c5 $m >> gpurun_out/motif_sweep.txt 2>&1
done
cat gpurun_out/motif_sweep.txt
