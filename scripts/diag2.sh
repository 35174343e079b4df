python scripts/diag_bench.py 2>&1 | head -2
nvidia-smi --query-gpu=clocks.sm --format=csv,noheader,nounits -lms 100 > /dev/null &
P=$!
python scripts/diag_bench.py 2>&1 | head -2
kill $P
