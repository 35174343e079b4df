export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_scoring.py tests/test_gpu_motifs.py -x -q -p no:cacheprovider 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_table2.py -x -q -p no:cacheprovider --durations=8 2>&1 | tail -25
