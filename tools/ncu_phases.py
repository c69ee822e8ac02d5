"""Per-phase stall breakdown of a cluster kernel from an ncu report (SASS page),
phases split at cluster barriers (UCGABAR_WAIT).

    python tools/ncu_phases.py <report.ncu-rep> [kernel-substring]
"""
import collections
import csv
import subprocess
import sys

STALLS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_lg", "stall_long_sb",
          "stall_math", "stall_mio", "stall_no_inst", "stall_not_selected", "stall_selected",
          "stall_short_sb", "stall_wait", "stall_misc", "stall_membar", "stall_drain", "stall_sleep"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    tot = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in data)
    cuts = [i for i, d in enumerate(data) if "UCGABAR_WAIT" in d["Source"]]
    prev = 0
    print(f"total samples {tot}")
    for c in cuts + [len(data)]:
        seg = data[prev:c + 1]
        s = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in seg)
        ex = sum(int(d["Instructions Executed"]) for d in seg)
        st = collections.Counter()
        for d in seg:
            for k in STALLS:
                v = d.get(k)
                if v and v != "-":
                    st[k] += int(v)
        top = ", ".join(f"{k[6:]} {100 * v / max(s, 1):.0f}%" for k, v in st.most_common(5))
        print(f"[{prev:5d},{c:5d}] {100 * s / tot:5.1f}% samples, {ex / 1e6:7.2f} M warp-instr | {top}")
        prev = c + 1


if __name__ == "__main__":
    main()
