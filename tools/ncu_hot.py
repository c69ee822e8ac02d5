"""Hottest SASS lines of an `ncu --page source --csv --print-source sass` export:
top instructions by warp stall samples and by executed instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = None
for i, r in enumerate(rows):
    if "Source" in r and any("Sampling" in c for c in r):
        hdr, body = r, rows[i + 1:]
        break
if hdr is None:
    print("no header found; first rows:", rows[:3])
    sys.exit(0)
col = {h: j for j, h in enumerate(hdr)}
samp = next(h for h in hdr if h.startswith("Warp Stall Sampling (All"))
exe = next((h for h in hdr if h.startswith("Instructions Executed")), None)


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


tot = sum(num(r[col[samp]]) for r in body if len(r) > col[samp])
print("columns:", [h for h in hdr][:40])
print("total stall samples", tot)
body.sort(key=lambda r: -num(r[col[samp]]) if len(r) > col[samp] else 0)
for r in body[:60]:
    print(f"{num(r[col[samp]]):8.0f} {100 * num(r[col[samp]]) / max(tot, 1):5.1f}%  "
          f"exe={num(r[col[exe]]) if exe else 0:12.0f}  {r[col['Source']][:90]}")

# instruction mix weighted by executed (warp-level) instructions
if exe:
    from collections import Counter

    mix = Counter()
    tot_exe = 0.0
    for r in body:
        if len(r) <= col[exe]:
            continue
        n = num(r[col[exe]])
        op = r[col["Source"]].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        mix[o.split(".")[0]] += n
        tot_exe += n
    print("\nexecuted warp instructions:", tot_exe)
    for o, n in mix.most_common(30):
        print(f"  {o:12s} {n:14.0f} {100 * n / max(tot_exe, 1):5.1f}%")
    print("\ntop lines by executed count:")
    body.sort(key=lambda r: -num(r[col[exe]]) if len(r) > col[exe] else 0)
    for r in body[:50]:
        print(f"exe={num(r[col[exe]]):12.0f}  {r[col['Source']][:100]}")
