# multi-layer launch: layer tests, attention suite, headline bench with/without the shared launch
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_layers_pdl_gpu.py -q -x 2>&1 | tail -25 > gpurun_out/layers_tests.log
timeout 300 python bench.py > gpurun_out/bench_layers.json 2> gpurun_out/bench_layers.err
KVMIX_LAYERS=0 timeout 300 python bench.py --no-e2e > gpurun_out/bench_nolayers.json 2> gpurun_out/bench_nolayers.err
timeout 300 python bench.py --config mistral-7b-32k > gpurun_out/bench_layers_mistral.json 2>> gpurun_out/bench_layers.err
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E  |FAILED|passed|failed|Error" | head -40 > gpurun_out/gpu_tests.log
