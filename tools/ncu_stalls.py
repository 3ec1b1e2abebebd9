"""Stall reasons and per-opcode stall samples of one kernel in an ncu report.

    python tools/ncu_stalls.py gpurun_out/x.ncu-rep [--top 30]
"""
import argparse
import csv
import io
import subprocess
from collections import Counter

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
d = {}
for h, v in zip(hdr, vals):
    if "smsp__average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
        d[h.split("stalled_")[1].replace("_per_issue_active.ratio", "")] = float(v)
    for key in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
                "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "launch__registers_per_thread"):
        if h == key:
            print(f"{key}: {v}")
print("stalls per issue:", ", ".join(f"{k} {v:.2f}" for k, v in
                                     sorted(d.items(), key=lambda x: -x[1])[:10]))
src = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iS]) for r in data if r[iS].isdigit())
c = Counter()
for r in data:
    if not r[iS].isdigit():
        continue
    parts = r[1].strip().split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") else parts[0]
    c[op.split(".")[0]] += int(r[iS])
print("samples by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in c.most_common(12)))
top = sorted((r for r in data if r[iS].isdigit()), key=lambda r: -int(r[iS]))[:a.top]
for r in top:
    print(f"  {r[0][-5:]} {int(r[iS]):7d}  {r[1].strip()[:80]}")
