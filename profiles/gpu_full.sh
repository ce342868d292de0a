mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  |FAILED|passed|failed|Error" | head -40 > gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for tool in synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python profiles/sanitize_drive.py > gpurun_out/${tool}_all.log 2>&1
done
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
