mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python profiles/sanitize_drive.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize/summary.txt
  tail -3 gpurun_out/sanitize/$tool.log >> gpurun_out/sanitize/summary.txt
done
