set -u
for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|========= (Invalid|Race|Barrier|Uninit)" gpurun_out/sanitize_$tool.log | head -8
  tail -2 gpurun_out/sanitize_$tool.log
done
