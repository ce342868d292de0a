"""Per-kernel launch counts, mean times and shares of the timed steps from an
`ncu --metrics gpu__time_duration.sum --csv` launch list (run HERE on the merged CSV).

  python profiles/launch_list.py gpurun_out/launches.csv LAST_N "command" > profiles/rNN_bench_launch_list.json
"""
import csv
import json
import re
import sys

path, last_n = sys.argv[1], int(sys.argv[2])
cmd = sys.argv[3] if len(sys.argv) > 3 else ""
with open(path) as f:
    rows = [r for r in csv.reader(line for line in f if line.startswith('"'))]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
launches = [(r[ki], float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1.0))
            for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
launches = launches[-last_n:]


def short(name):
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(.*$", "", name)
    return re.sub(r"(\w+::)*<?unnamed>?::", "", name)


tot = sum(t for _, t in launches)
agg = {}
for n, t in launches:
    a = agg.setdefault(short(n), [0, 0.0])
    a[0] += 1
    a[1] += t
out = {"command": cmd,
       "note": f"last {last_n} launches (the timed steps); cold-cache serialized per-launch times: only the SHARE is comparable",
       "kernels": {k: {"launches": c, "mean_us": s / c, "share": s / tot} for k, (c, s) in sorted(agg.items(), key=lambda x: -x[1][1])}}
print(json.dumps(out, indent=1))
