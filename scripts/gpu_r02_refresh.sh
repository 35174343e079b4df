# launch list of config 4 (diamond, apex S) for traffic.json
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4-diamond.csv python scripts/prof_step.py c4-diamond 1 > gpurun_out/prof_c4d.txt 2>&1
tail -3 gpurun_out/prof_c4d.txt
