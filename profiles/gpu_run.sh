mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
KVMIX_WS=2 timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench_ws2.json 2> gpurun_out/bench_ws2.err
KVMIX_WS=0 timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench_ws0.json 2> gpurun_out/bench_ws0.err
timeout 600 python bench.py --config mistral-7b-32k --no-e2e --no-cpu > gpurun_out/bench_mistral.json 2> gpurun_out/bench_mistral.err
tail -3 gpurun_out/*.log gpurun_out/*.json
