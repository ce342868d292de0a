# per-source-line instruction / stall profile of configs[1]'s two tier launches (K3V4 and K2V2, one query row)
O=gpurun_out/lines_c1
mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attend_mma_layers -s 6 -c 2 \
  -o $O/prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-check > $O/prof.log 2>&1
python profiles/ncu_lines.py $O/prof.ncu-rep '(int)128, (int)2, (int)2, (int)1' 70 > $O/lines_k2v2.txt 2>&1
python profiles/ncu_lines.py $O/prof.ncu-rep '(int)128, (int)2, (int)2, (int)1' 40 stall > $O/lines_k2v2_stall.txt 2>&1
python profiles/ncu_lines.py $O/prof.ncu-rep '(int)128, (int)3, (int)4, (int)1' 60 > $O/lines_k3v4.txt 2>&1
rm -f $O/prof.ncu-rep
for i in 1 2; do timeout 300 python bench.py --config layer-4k --no-cpu > $O/bench_layer-4k_$i.json 2>> $O/bench.err; done
KVMIX_R4=0 timeout 300 python bench.py --config layer-4k --no-cpu > $O/bench_layer-4k_r4off.json 2>> $O/bench.err
