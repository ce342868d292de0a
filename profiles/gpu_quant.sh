mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "quant or cache or pack or mixed3 or export" 2>&1 | tail -5 > gpurun_out/quant_tests.log
timeout 600 python bench.py --config quant-sweep > gpurun_out/bench_quant.json 2> gpurun_out/bench_quant.err
