mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1000 python -m pytest tests/test_gpu_checked.py -x -q -p no:cacheprovider > gpurun_out/gputest_checked.txt 2>&1
tail -15 gpurun_out/gputest_checked.txt
