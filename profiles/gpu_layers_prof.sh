# ncu evidence for the multi-layer launch: launch list of 32 timed steps (one Key age-out
# step included) and one full capture of each tier's launch of the first timed step
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/layers_launches.csv \
  python bench.py --steps 32 --warmup 3 --no-e2e --no-cpu --no-check > gpurun_out/layers_launches_bench.json 2> gpurun_out/layers_launches.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attend_mma_layers -s 6 -c 2 \
  -o gpurun_out/layers_prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-check > gpurun_out/layers_prof.log 2>&1
