mkdir -p gpurun_out
timeout 240 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_table<\(int\)0' -s 1 -c 1 -o gpurun_out/prof_m7c python scripts/prof_motif.py c5 M2,M7 2 > gpurun_out/ncu_m7c.log 2>&1
timeout 240 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_table<\(int\)2' -s 5 -c 1 -o gpurun_out/prof_m7s python scripts/prof_motif.py c5 M2,M7 2 > gpurun_out/ncu_m7s.log 2>&1
ls gpurun_out/*.ncu-rep
