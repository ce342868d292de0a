# four-row passes, round 3: beta reduction + hoisted Value scale, shuffled p (pbuf reverted); K3 R4 at 12 warps as the alternative
mkdir -p gpurun_out/r4c
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_bench_shapes_gpu.py tests/test_layers_pdl_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r4c/tests.log
for i in 1 2; do
  timeout 300 python bench.py --config mistral-7b-32k --no-cpu --no-e2e > gpurun_out/r4c/mistral_def_$i.json 2>> gpurun_out/r4c/bench.err
  KVMIX_LIB=$PWD/paper_2506_08018_b200/libkvmix_ab16.so timeout 300 python bench.py --config mistral-7b-32k --no-cpu --no-e2e > gpurun_out/r4c/mistral_k3w12_$i.json 2>> gpurun_out/r4c/bench.err
done
KVMIX_R4=0 timeout 300 python bench.py --config mistral-7b-32k --no-cpu --no-e2e > gpurun_out/r4c/mistral_r2.json 2>> gpurun_out/r4c/bench.err
