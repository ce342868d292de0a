# Mixed3 Value quantizer with the group fold from the staging registers: quant parity + sweep
O=gpurun_out/m3v7
mkdir -p $O
timeout 900 python -m pytest tests/test_quant_gpu.py tests/test_cache_gpu.py -m gpu -q -x 2>&1 | tail -3 > $O/tests.log
for i in 1 2; do timeout 600 python bench.py --config quant-sweep --no-cpu --no-e2e > $O/sweep_$i.json 2>> $O/bench.err; done
