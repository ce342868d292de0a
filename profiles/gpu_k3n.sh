# narrow-slot field table read through a funnel shift (K3 layers): parity subset + configs[1] / configs[2]
mkdir -p gpurun_out/k3n
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_bench_shapes_gpu.py tests/test_layers_pdl_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/k3n/tests.log
for i in 1 2; do
  timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/k3n/llama_$i.json 2>> gpurun_out/k3n/bench.err
  timeout 300 python bench.py --config mistral-7b-32k --no-cpu --no-e2e > gpurun_out/k3n/mistral_$i.json 2>> gpurun_out/k3n/bench.err
done
