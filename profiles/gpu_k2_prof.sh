# ncu of the Mixed3 Value quantizer (3-bit Values, gs 32 and 128) on the sweep shape, line profile on the box
O=gpurun_out/k2
mkdir -p $O
cat > $O/drive.py <<'PY'
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2506_08018_b200 as K
x = torch.randn(16, 32, 4096, 128, device="cuda", dtype=torch.float16)
for gs in (32,):
    for _ in range(2):
        K.quantize_key_tensor(x, K.QuantSpec(2, K.Grouping(0), gs))
torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quantize_key -s 1 -c 1 -o $O/prof python $O/drive.py > $O/prof.log 2>&1
python profiles/ncu_summary.py $O/prof.ncu-rep --json $O/ncu_summary.json > $O/ncu_summary.txt 2>&1
python profiles/ncu_lines.py $O/prof.ncu-rep '2, (int)128>' 50 > $O/lines_gs32.txt 2>&1
python profiles/ncu_lines.py $O/prof.ncu-rep '2, (int)128>' 30 stall > $O/lines_gs32_stall.txt 2>&1
python profiles/ncu_lines.py $O/prof.ncu-rep '2, (int)128>' 40 > $O/lines_gs128.txt 2>&1
ncu -i $O/prof.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
rm -f $O/prof.ncu-rep
