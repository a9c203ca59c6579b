"""Summarise an `ncu --set full` report of one bench step into profiles/ JSON + text.

usage: python tools/ncu_summary.py report.ncu-rep out_prefix [config]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

rep, out = sys.argv[1], sys.argv[2]
cfg = sys.argv[3] if len(sys.argv) > 3 else "C1"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = {
    "time_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
}
units = rows[1]
def val(row, key):
    i = hdr.index(want[key]) if want[key] in hdr else -1
    if i < 0 or not row[i]:
        return None
    v = float(row[i].replace(",", ""))
    u = units[i]
    if key.startswith("dram_") and key != "dram_pct":
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    if key == "time_us":
        v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
    return v
kern = []
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0]
    name = name.replace("spava::", "").replace("unnamed>::", "").strip(":")
    kern.append({"kernel": name, **{k: val(r, k) for k in want}})
agg = defaultdict(lambda: defaultdict(float))
for k in kern:
    a = agg[k["kernel"]]
    a["launches"] += 1
    for f in ("time_us", "dram_read", "dram_write"):
        a[f] += k[f] or 0
summary = {"config": cfg, "launches": kern, "per_kernel": {}}
for name, a in agg.items():
    n = a["launches"]
    summary["per_kernel"][name] = {"launches": n, "time_us": a["time_us"],
                                   "dram_bytes_per_launch": (a["dram_read"] + a["dram_write"]) / n}
attn = summary["per_kernel"].get("attn_fwd_kernel")
summary[cfg] = {"dram_bytes_per_launch": attn["dram_bytes_per_launch"] if attn else None}
json.dump(summary, open(out + ".json", "w"), indent=1)
with open(out + ".txt", "w") as f:
    f.write(f"ncu --set full, one bench step ({cfg}); cold-cache serialized replays\n")
    f.write(f"{'kernel':22s} {'us':>9s} {'DRAM MB':>9s} {'tensor%':>8s} {'xu%':>6s} {'fma%':>6s} {'fp64%':>6s} {'issue%':>7s} {'dram%':>6s} {'l2%':>6s} {'l1%':>6s} regs grid\n")
    for k in kern:
        f.write(f"{k['kernel'][:22]:22s} {k['time_us']:9.1f} {((k['dram_read'] or 0)+(k['dram_write'] or 0))/1e6:9.1f} "
                f"{k['tensor_pipe_pct'] or 0:8.1f} {k['xu_pct'] or 0:6.1f} {k['fma_pct'] or 0:6.1f} {k['fp64_pct'] or 0:6.1f} "
                f"{k['issue_pct'] or 0:7.1f} {k['dram_pct'] or 0:6.1f} {k['l2_pct'] or 0:6.1f} {k['l1_pct'] or 0:6.1f} "
                f"{int(k['regs'] or 0):4d} {int(k['grid'] or 0)}\n")
print(open(out + ".txt").read())
