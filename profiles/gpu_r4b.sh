# four-row passes, round 2: parity subset, configs[2] bench (default vs 16-warp register budget), configs[1] bench
mkdir -p gpurun_out/r4b
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_bench_shapes_gpu.py tests/test_layers_pdl_gpu.py tests/test_graph_gpu.py tests/test_attention_tc_gpu.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r4b/tests.log
for i in 1 2; do
  timeout 300 python bench.py --config mistral-7b-32k --no-cpu --no-e2e > gpurun_out/r4b/mistral_def_$i.json 2>> gpurun_out/r4b/bench.err
  KVMIX_LIB=$PWD/paper_2506_08018_b200/libkvmix_ab16.so timeout 300 python bench.py --config mistral-7b-32k --no-cpu --no-e2e > gpurun_out/r4b/mistral_w16_$i.json 2>> gpurun_out/r4b/bench.err
done
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/r4b/llama_def.json 2>> gpurun_out/r4b/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_mma_layers -s 6 -c 2 \
  -o gpurun_out/r4b/prof python bench.py --config mistral-7b-32k --steps 1 --warmup 3 --no-e2e --no-cpu --no-check > gpurun_out/r4b/prof.log 2>&1
python profiles/ncu_summary.py gpurun_out/r4b/prof.ncu-rep --json gpurun_out/r4b/ncu_summary.json > gpurun_out/r4b/ncu_summary.txt 2>&1
python profiles/ncu_lines.py gpurun_out/r4b/prof.ncu-rep '(int)128, (int)2, (int)2, (int)4' 70 > gpurun_out/r4b/lines_k2v2.txt 2>&1
python profiles/ncu_lines.py gpurun_out/r4b/prof.ncu-rep '(int)128, (int)2, (int)2, (int)4' 40 stall > gpurun_out/r4b/lines_k2v2_stall.txt 2>&1
python profiles/ncu_lines.py gpurun_out/r4b/prof.ncu-rep '(int)128, (int)3, (int)4, (int)4' 50 > gpurun_out/r4b/lines_k3v4.txt 2>&1
rm -f gpurun_out/r4b/prof.ncu-rep
