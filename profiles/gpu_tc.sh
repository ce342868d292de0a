mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_attention_tc_gpu.py -x -q 2>&1 | tail -30 > gpurun_out/tc_tests.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err
KVMIX_TC=0 timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_notc.json 2> gpurun_out/bench_notc.err
timeout 300 python bench.py --config mistral-7b-32k --no-cpu --no-e2e > gpurun_out/bench_mistral_tc.json 2> gpurun_out/bench_mistral_tc.err
