# round-end evidence after the last quantizer changes (profiles/r2/final5/): full GPU suite, smoke,
# the headline bench line and the quantize/pack sweep
O=gpurun_out/final5
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  |FAILED|passed|failed|Error" | head -40 > $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 300 python bench.py > $O/bench_llama2-7b-8k.json 2> $O/bench.err
timeout 600 python bench.py --config quant-sweep > $O/bench_quant_sweep.json 2>> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_quant.csv \
  python bench.py --config quant-sweep --steps 2 --warmup 3 --no-e2e --no-cpu --no-check > $O/launches_quant_bench.json 2>> $O/ncu.err
