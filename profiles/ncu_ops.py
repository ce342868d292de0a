"""SASS opcode histogram (instructions executed) of one kernel in an ncu report.

  python profiles/ncu_ops.py gpurun_out/prof.ncu-rep '(int)128, (int)2, (int)2' [per_unit]
"""
import collections
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
per = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
cnt, fn, hdr, tot = collections.Counter(), None, None, 0
stall = collections.Counter()
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "Kernel Name":
        fn = r[1]
    elif r and r[0] == "Address":
        hdr = r
    elif fn and pat in fn and hdr and r and r[0].startswith("0x"):
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        ins = r[1].strip().split()
        if not ins:
            continue
        op = ins[0]
        if op.startswith("@"):
            op = ins[1]
        op = op.rstrip(";")
        n = float(r[ie] or 0)
        cnt[op] += n
        stall[op] += float(r[ss] or 0)
        tot += n
st = sum(stall.values()) or 1
print(f"total {tot:.4g}  per unit {tot / per:.1f}")
for op, n in cnt.most_common(45):
    print(f"{op:28s} {n / per:9.1f} {100 * n / tot:5.1f}%  stall {100 * stall[op] / st:5.1f}%")
