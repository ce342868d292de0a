"""Per-CUDA-source-line instruction / stall totals of one kernel in an ncu report.

  python profiles/ncu_lines.py gpurun_out/prof.ncu-rep '(int)128, (int)2, (int)2' [N]
"""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
by_stall = len(sys.argv) > 4 and sys.argv[4] == "stall"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
lines, fn, hdr, path = [], None, None, None


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        path = r[1]
    elif len(r) == 2 and r[0] == "Function Name":
        fn = r[1]
    elif r and r[0] == "Line No":
        hdr = r
    elif fn and pat in fn and hdr and r and r[0] not in ("", "-"):
        ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        lines.append((num(r[ie]), num(r[ss]), path.split("/")[-1], r[0], r[1].strip()[:90]))
tot = sum(x[0] for x in lines) or 1
tots = sum(x[1] for x in lines) or 1
print(f"total inst {tot:.4g}")
for n, s, f, ln, src in sorted(lines, key=lambda x: x[1] if by_stall else x[0], reverse=True)[:top]:
    print(f"{100*n/tot:5.1f}% inst {100*s/tots:5.1f}% stall  {f}:{ln:>4}  {src}")
