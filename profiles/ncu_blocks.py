"""Per-basic-block instruction/stall breakdown of one kernel in an ncu report (SASS page).

  python profiles/ncu_blocks.py gpurun_out/prof.ncu-rep 'attend_mma_kernel<(int)128, (int)2'
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
secs, cur = [], None
for r in rows:
    if len(r) >= 2 and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        secs.append(cur)
        continue
    if r and r[0] == "Address":
        cur["hdr"] = r
        continue
    if cur is not None and len(r) > 5:
        cur["rows"].append(r)
for s in secs:
    if pat not in s["name"]:
        continue
    h = s["hdr"]
    ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    R = s["rows"]
    tot = sum(float(r[ie] or 0) for r in R)
    tots = sum(float(r[ss] or 0) for r in R)
    cnt, stl, ops = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    for r in R:
        n = float(r[ie] or 0)
        cnt[n] += 1
        stl[n] += float(r[ss] or 0)
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[1])
        if m:
            ops[n][m.group(2)] += 1
    print(s["name"][:100], f"total inst {tot:.3e}")
    for n, c in sorted(cnt.items(), key=lambda x: -x[0] * x[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 8]:
        print(f"exec {n:10.0f} x {c:5d} = {n * c / tot * 100:5.1f}% inst, {stl[n] / tots * 100:5.1f}% stalls  "
              f"{dict(ops[n].most_common(10))}")
    break
