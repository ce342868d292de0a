# A/B of an alternative build (KVMIX_LIB) against the default library: 2 bench runs each
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu $BENCH_ARGS > gpurun_out/ab_def_$i.json 2>> gpurun_out/ab.err
  KVMIX_LIB=$PWD/$1 timeout 300 python bench.py --no-e2e --no-cpu $BENCH_ARGS > gpurun_out/ab_alt_$i.json 2>> gpurun_out/ab.err
done
KVMIX_LIB=$PWD/$1 timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_layers_pdl_gpu.py -q -x 2>&1 | tail -2 > gpurun_out/ab_alt_tests.log
