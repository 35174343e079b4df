# final verification of the committed build: the GPU suite + smoke (what the driver runs)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_verify.txt 2>&1
tail -2 gpurun_out/gputest_verify.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
