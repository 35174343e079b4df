mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_motifs.py -q -p no:cacheprovider -k "two_chunk" > gpurun_out/gputest_t.txt 2>&1
tail -15 gpurun_out/gputest_t.txt
