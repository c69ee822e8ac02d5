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
