# GQA four-row passes (R = 4): parity subset + configs[2] A/B (KVMIX_R4 = 1 vs 0)
mkdir -p gpurun_out/r4
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_bench_shapes_gpu.py tests/test_layers_pdl_gpu.py tests/test_graph_gpu.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r4/tests.log
timeout 300 python bench.py --config mistral-7b-32k --no-cpu > gpurun_out/r4/bench_mistral_r4.json 2> gpurun_out/r4/bench.err
KVMIX_R4=0 timeout 300 python bench.py --config mistral-7b-32k --no-cpu > gpurun_out/r4/bench_mistral_r2.json 2>> gpurun_out/r4/bench.err
timeout 300 python bench.py --config mistral-7b-32k --no-cpu > gpurun_out/r4/bench_mistral_r4b.json 2>> gpurun_out/r4/bench.err
