# r02: motif-table tests first (new code), then the rest of the GPU suite, then benches per motif set
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_motifs.py -x -q -p no:cacheprovider > gpurun_out/gputest_motifs.txt 2>&1
tail -30 gpurun_out/gputest_motifs.txt
for m in all heavy-hex M2,M5 M2,M3,M6 M2,M7 M2,M3,M8; do
  timeout 300 python scripts/motif_bench.py c5 $m >> gpurun_out/motif_bench.txt 2>&1
done
cat gpurun_out/motif_bench.txt
