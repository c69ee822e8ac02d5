#!/usr/bin/env python
"""Print the key sections of an ncu --page details CSV (tools/ncu_capture.sh)."""
import csv
import sys

KEEP = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
        "Warp State Statistics", "Occupancy", "Launch Statistics")
NAMES = ("Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
         "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Memory Throughput",
         "Warp Cycles Per Issued Instruction", "Achieved Active Warps Per SM", "Registers Per Thread",
         "Theoretical Occupancy", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
         "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Pipes Busy")


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Section Name") in KEEP and d.get("Metric Name") in NAMES:
            print(f"  {d['Metric Name'][:42]:42s} {d['Metric Value']} {d.get('Metric Unit', '')}")
    # pipe utilisation and stall reasons from the raw page, if present
    raw = path.replace("_details.csv", "_raw.csv")
    try:
        rr = list(csv.reader(open(raw)))
    except OSError:
        return
    h, units, vals = rr[0], rr[1], rr[2]
    for name, u, v in zip(h, units, vals):
        if (name.startswith("sm__inst_executed_pipe_") and name.endswith("pct_of_peak_sustained_active")) or \
           (name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio")) or \
           name.startswith("l1tex__data_bank_conflicts_pipe_lsu_mem_shared") or \
           name.startswith("l1tex__data_pipe_lsu_wavefronts_mem_shared") or \
           name in ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum",
                    "dram__bytes_read.sum", "dram__bytes_write.sum"):
            try:
                if float(v.replace(",", "")) == 0:
                    continue
            except ValueError:
                pass
            print(f"  {name[:78]:78s} {v} {u}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("=====", p)
        main(p)
