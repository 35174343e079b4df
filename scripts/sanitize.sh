# compute-sanitizer memcheck / racecheck / initcheck / synccheck over scripts/sanitize_cases.py
# (SURVEY §5); summaries -> gpurun_out/sanitize_*.txt (copied to profiles/ when judged).
mkdir -p gpurun_out
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -4 gpurun_out/sanitize_$tool.txt
done
