# ncu full capture of one launch per quantize setting (bench.py --config quant-sweep)
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:quantize_key -s 27 -c 3 \
  -o gpurun_out/quant_prof python bench.py --config quant-sweep --steps 1 --warmup 3 --no-e2e --no-cpu --no-check > gpurun_out/quant_prof.log 2>&1
