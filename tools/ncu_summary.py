#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (committed evidence).

  tools/ncu_summary.py launches <launches.csv> <out.md>        per-kernel share of a step
  tools/ncu_summary.py full <prof.ncu-rep> <out.md> [traffic.json workload]
"""
import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_shared_mem",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")) / 1e3)
    tot = sum(sum(v) / len(v) for v in agg.values())
    lines = [f"# ncu launch list: {path}", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised; compare shares)", "",
             "| kernel | launches | mean us | share of step |", "|---|---|---|---|"]
    for k, v in agg.items():
        m = sum(v) / len(v)
        lines.append(f"| {k} | {len(v)} | {m:.2f} | {100 * m / tot:.1f} % |")
    lines.append(f"| **sum of means** | | {tot:.2f} | |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(path, out, traffic_json=None, workload=None):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"]).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full summary: {path}", ""]
    traffic = {}
    for r in data:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "")
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"| {m} | {r[i]} | {units[i]} |")
        lines.append("")
        try:
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            u1 = units[hdr.index("dram__bytes_read.sum")]
            u2 = units[hdr.index("dram__bytes_write.sum")]
            key = short.split("<")[0].replace("k_", "")
            traffic.setdefault(key, rd * scale.get(u1, 1) + wr * scale.get(u2, 1))
        except (ValueError, KeyError):
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json and workload:
        try:
            d = json.load(open(traffic_json))
        except (OSError, ValueError):
            d = {}
        d[workload] = traffic
        json.dump(d, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], *(sys.argv[4:6]))
