# ncu evidence for configs[2] with four-row passes: launch list + one full capture of each tier's launch
mkdir -p gpurun_out/r4p
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4p/launches.csv \
  python bench.py --config mistral-7b-32k --steps 32 --warmup 3 --no-e2e --no-cpu --no-check > gpurun_out/r4p/launches_bench.json 2> gpurun_out/r4p/launches.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attend_mma_layers -s 6 -c 2 \
  -o gpurun_out/r4p/prof python bench.py --config mistral-7b-32k --steps 1 --warmup 3 --no-e2e --no-cpu --no-check > gpurun_out/r4p/prof.log 2>&1
# summarise on the box (the full reports exceed the copy-back limit)
python profiles/ncu_summary.py gpurun_out/r4p/prof.ncu-rep --json gpurun_out/r4p/ncu_summary.json > gpurun_out/r4p/ncu_summary.txt 2>&1
ncu -i gpurun_out/r4p/prof.ncu-rep --page source --csv --print-source sass > gpurun_out/r4p/source.csv 2>/dev/null
ls -la gpurun_out/r4p > gpurun_out/r4p/ls.txt
gzip -f gpurun_out/r4p/source.csv
rm -f gpurun_out/r4p/prof.ncu-rep
