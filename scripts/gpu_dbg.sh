export PYTHONUNBUFFERED=1
timeout 300 python -X faulthandler -m pytest tests/test_gpu_motifs.py -x -v -p no:cacheprovider --timeout 60 -k "lattices" 2>&1 | tail -60
