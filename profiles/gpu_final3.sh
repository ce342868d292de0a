# round-end evidence after the four-row GQA passes (profiles/r2/final3/): full GPU suite, smoke,
# every bench config, launch list + full ncu capture of both tier launches (configs[1] and [2])
O=gpurun_out/final3
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  |FAILED|passed|failed|Error" | head -40 > $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 300 python bench.py > $O/bench_llama2-7b-8k.json 2> $O/bench.err
timeout 300 python bench.py --config mistral-7b-32k > $O/bench_mistral-7b-32k.json 2>> $O/bench.err
timeout 300 python bench.py --config layer-4k > $O/bench_layer-4k.json 2>> $O/bench.err
timeout 600 python bench.py --config llama2-13b-128k-shard > $O/bench_llama2-13b-128k-shard.json 2>> $O/bench.err
timeout 600 python bench.py --config quant-sweep > $O/bench_quant_sweep.json 2>> $O/bench.err
for C in llama2-7b-8k mistral-7b-32k; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$C.csv \
    python bench.py --config $C --steps 32 --warmup 3 --no-e2e --no-cpu --no-check > $O/launches_bench_$C.json 2>> $O/ncu.err
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attend_mma_layers -s 6 -c 2 \
    -o $O/prof_$C python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu --no-check > $O/prof_$C.log 2>&1
  python profiles/ncu_summary.py $O/prof_$C.ncu-rep --json $O/ncu_summary_$C.json > $O/ncu_summary_$C.txt 2>&1
  rm -f $O/prof_$C.ncu-rep
done
