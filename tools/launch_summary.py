"""Mean per-kernel duration from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

for fn in sys.argv[1:]:
    print("==", fn)
    rows = [r for r in csv.reader(open(fn)) if len(r) > 10]
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    d = collections.OrderedDict()
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        d.setdefault(r[idx["Kernel Name"]][:70], []).append(float(r[idx["Metric Value"]]))
    for n, v in d.items():
        print(f"{n:70s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.1f} us")
