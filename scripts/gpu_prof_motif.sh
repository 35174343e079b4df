mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_table" -s 8 -c 2 -o gpurun_out/prof_m7 python scripts/prof_motif.py c5 M2,M7 3 > gpurun_out/ncu_m7.log 2>&1
tail -3 gpurun_out/ncu_m7.log
ncu -i gpurun_out/prof_m7.ncu-rep --page details --csv > gpurun_out/prof_m7_details.csv 2>&1
ls -la gpurun_out/
