mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 400 python -m pytest tests/test_gpu_motifs.py -x -q -p no:cacheprovider > gpurun_out/gputest_motifs.txt 2>&1
tail -3 gpurun_out/gputest_motifs.txt
rm -f gpurun_out/motif_bench.txt
for m in M2,M7 M2,M3,M8 M2,M3,M6; do
  timeout 60 python scripts/motif_bench.py c5 $m >> gpurun_out/motif_bench.txt 2>&1
done
cat gpurun_out/motif_bench.txt
timeout 240 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_table<\(int\)0" -s 1 -c 1 -o gpurun_out/prof_m7c python scripts/prof_motif.py c5 M2,M7 2 > gpurun_out/ncu_m7c.log 2>&1
timeout 240 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_table<\(int\)2" -s 5 -c 1 -o gpurun_out/prof_m7s python scripts/prof_motif.py c5 M2,M7 2 > gpurun_out/ncu_m7s.log 2>&1
tail -2 gpurun_out/ncu_m7c.log gpurun_out/ncu_m7s.log
