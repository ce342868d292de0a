mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  |FAILED|passed|failed|Error" | head -40 > gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --config layer-4k > gpurun_out/bench_layer4k.json 2>> gpurun_out/bench_default.err
timeout 600 python bench.py --config llama2-13b-128k-shard > gpurun_out/bench_13b.json 2>> gpurun_out/bench_default.err
