"""Pick metrics (substring match) from an `ncu --page raw --csv` export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
pats = sys.argv[2:]
for h, u, v in zip(hdr, units, vals):
    if any(p in h for p in pats):
        print(f"{h:90s} {v:>20s} {u}")
