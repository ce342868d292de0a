"""Summarise an ncu report (run HERE, not on the GPU box): per kernel duration, DRAM bytes,
achieved DRAM GB/s, instructions, issue-slot use and the top warp-stall reasons.

  python profiles/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: v for h, v in zip(hdr, r)}
        u = {h: v for h, v in zip(hdr, units)}
        res.append((d, u))
    return res


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def scale(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
         "msecond": 1e-3, "s": 1, "nsecond": 1e-9}.get(unit, 1)
    return v * f


def summarize(rep):
    out = []
    for d, u in raw(rep):
        k = {"kernel": d.get("Kernel Name", "")[:120]}
        dur = scale(num(d.get("gpu__time_duration.sum")), u.get("gpu__time_duration.sum"))
        rd = scale(num(d.get("dram__bytes_read.sum")), u.get("dram__bytes_read.sum"))
        wr = scale(num(d.get("dram__bytes_write.sum")), u.get("dram__bytes_write.sum"))
        k.update(duration_us=dur * 1e6, dram_read_MB=rd / 1e6, dram_write_MB=wr / 1e6,
                 dram_GBps=(rd + wr) / dur / 1e9,
                 inst_executed=num(d.get("smsp__inst_executed.sum")),
                 issue_active_pct=num(d.get("sm__inst_issued.avg.pct_of_peak_sustained_active")),
                 dram_pct_of_peak=num(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")),
                 regs=num(d.get("launch__registers_per_thread")),
                 achieved_occupancy_pct=num(d.get("sm__warps_active.avg.pct_of_peak_sustained_active")))
        st = []
        for key, v in d.items():
            if key.startswith("smsp__average_warps_issue_stalled_") and key.endswith("_per_issue_active.ratio"):
                x = num(v)
                if x is not None:
                    st.append((x, key[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        k["top_stalls"] = [(n, round(x, 3)) for x, n in sorted(st, reverse=True)[:6]]
        out.append(k)
    return out


if __name__ == "__main__":
    s = summarize(sys.argv[1])
    for k in s:
        print(json.dumps(k))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(s, f, indent=1)
