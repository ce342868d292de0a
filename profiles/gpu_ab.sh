# headline A/B: three default bench runs (no e2e) for noise, plus the layer tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_layers_pdl_gpu.py tests/test_attention_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/ab_tests.log
for i in 1 2 3; do timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/ab_$i.json 2>> gpurun_out/ab.err; done
