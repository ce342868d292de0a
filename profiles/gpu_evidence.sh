mkdir -p gpurun_out/ev
O=gpurun_out/ev
timeout 400 python bench.py > $O/bench_llama2-7b-8k.json 2> $O/b1.err
timeout 400 python bench.py --config mistral-7b-32k > $O/bench_mistral-7b-32k.json 2> $O/b2.err
timeout 400 python bench.py --config layer-4k > $O/bench_layer-4k.json 2> $O/b3.err
timeout 600 python bench.py --config llama2-13b-128k-shard --no-cpu --steps 10 --warmup 3 > $O/bench_llama2-13b-128k-shard.json 2> $O/b4.err
timeout 600 python bench.py --config quant-sweep > $O/bench_quant_sweep.json 2> $O/b5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm.json 2> $O/b6.err
timeout 400 python profiles/attend_time.py > $O/attend_time_mha.txt 2>&1
KVMIX_TC=1 timeout 400 python profiles/attend_time.py > $O/attend_time_mha_tc.txt 2>&1
SHAPE=8,8,4,32768 timeout 400 python profiles/attend_time.py > $O/attend_time_gqa.txt 2>&1
KVMIX_TC=1 SHAPE=8,8,4,32768 timeout 400 python profiles/attend_time.py > $O/attend_time_gqa_tc.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-check > $O/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 1 -c 2 -o $O/mma_prof python profiles/drive_attend.py > $O/ncu1.log 2>&1
KVMIX_TC=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_tc -s 1 -c 1 -o $O/tc_prof python profiles/drive_attend.py 0 > $O/ncu2.log 2>&1
