mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "quant" 2>&1 | tail -1 > gpurun_out/quant_tests.log
timeout 600 python bench.py --config quant-sweep --no-e2e --no-cpu > gpurun_out/bq_a.json 2> /dev/null
KVMIX_QK_TOK=128 KVMIX_QK_THREADS=256 timeout 600 python bench.py --config quant-sweep --no-e2e --no-cpu > gpurun_out/bq_b.json 2> /dev/null
KVMIX_QK_TOK=32 KVMIX_QK_THREADS=64 timeout 600 python bench.py --config quant-sweep --no-e2e --no-cpu > gpurun_out/bq_c.json 2> /dev/null
KVMIX_QK_TOK=128 KVMIX_QK_THREADS=128 timeout 600 python bench.py --config quant-sweep --no-e2e --no-cpu > gpurun_out/bq_d.json 2> /dev/null
