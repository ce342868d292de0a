# sanitizers over the multi-layer section only (SANITIZE_CONFIGS picks one single-layer config)
mkdir -p gpurun_out/sanitize_layers
for tool in memcheck racecheck synccheck initcheck; do
  SANITIZE_CONFIGS=0 timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python profiles/sanitize_drive.py > gpurun_out/sanitize_layers/$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_layers/summary.txt
  tail -3 gpurun_out/sanitize_layers/$tool.log >> gpurun_out/sanitize_layers/summary.txt
done
