mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_motifs.py -x -q -p no:cacheprovider > gpurun_out/gputest_motifs.txt 2>&1
tail -3 gpurun_out/gputest_motifs.txt
timeout 1500 python -m pytest tests/test_gpu_table2.py -q -p no:cacheprovider --durations=10 -k "not grid60-100" > gpurun_out/gputest_t2.txt 2>&1
tail -15 gpurun_out/gputest_t2.txt
