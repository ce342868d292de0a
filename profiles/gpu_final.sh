# round-end evidence: full GPU suite, smoke, every bench config (profiles/r2/final/)
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  |FAILED|passed|failed|Error" | head -40 > gpurun_out/final/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/final/bench_llama2-7b-8k.json 2> gpurun_out/final/bench.err
timeout 300 python bench.py --config mistral-7b-32k > gpurun_out/final/bench_mistral-7b-32k.json 2>> gpurun_out/final/bench.err
timeout 300 python bench.py --config layer-4k > gpurun_out/final/bench_layer-4k.json 2>> gpurun_out/final/bench.err
timeout 600 python bench.py --config llama2-13b-128k-shard > gpurun_out/final/bench_llama2-13b-128k-shard.json 2>> gpurun_out/final/bench.err
timeout 600 python bench.py --config quant-sweep > gpurun_out/final/bench_quant_sweep.json 2>> gpurun_out/final/bench.err
