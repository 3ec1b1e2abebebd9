"""Summarise an ncu --set full report (and optionally a launch-list CSV) into profiles/*.json.

    python tools/ncu_summary.py gpurun_out/k1s_c2_r01.ncu-rep --launches gpurun_out/launches_c2.csv \
        --variant "<kernel variant name>" --out profiles/ncu_k1_c2_r01.json
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefronts_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
              "ms": 1e-3, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--launches")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    hdr, units, rows = raw(a.rep)
    kernels = []
    for v in rows:
        d = {"kernel": v[hdr.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                val = v[i].replace(",", "")
                try:
                    x = float(val) * UNIT_SCALE.get(units[i], 1.0)
                except ValueError:
                    continue
                d[name] = x
        stalls = []
        for i, k in enumerate(hdr):
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v[i]), k.split("stalled_")[1].split("_per_issue")[0]))
                except ValueError:
                    pass
        d["top_stalls_per_issue"] = {n: round(s, 3) for s, n in sorted(stalls, reverse=True)[:6]}
        if "dram_read" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d.get("dram_write", 0.0)
        kernels.append(d)
    summary = {"report": a.rep, "variant": a.variant, "kernels": kernels}
    if kernels and "dram_bytes_per_launch" in kernels[0]:
        summary["dram_bytes_per_launch"] = kernels[0]["dram_bytes_per_launch"]
    if a.launches:
        lrows = list(csv.reader(open(a.launches)))
        start = next(i for i, r in enumerate(lrows) if r and r[0] == "ID")
        h = lrows[start]
        ni, vi = h.index("Kernel Name"), h.index("Metric Value")
        launches = [(r[ni].split("(")[0], float(r[vi].replace(",", ""))) for r in lrows[start + 1:]
                    if len(r) > vi]
        import re
        ours = re.compile(r"(mcp::|\bk1|\bk5|\bk_)")
        mine = [(n, t) for n, t in launches if ours.search(n)]
        tot = sum(t for _, t in mine)
        agg = {}
        for n, t in mine:
            agg.setdefault(n, []).append(t)
        summary["launch_list_ns"] = {n: {"count": len(ts), "mean_ns": sum(ts) / len(ts),
                                          "share_of_mcp_time": sum(ts) / tot}
                                     for n, ts in agg.items()}
    json.dump(summary, open(a.out, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
