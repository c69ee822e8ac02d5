"""Print the key numbers of bench.py JSON lines (files given on the command line)."""
import json
import sys

for fn in sys.argv[1:]:
    print("==", fn)
    for line in open(fn):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        print({k: d.get(k) for k in ("impl", "value", "ms_per_step", "pipeline", "n_gpus", "scaling",
                                     "gpu_launches", "steps_timed")})
        r = d.get("roofline")
        if r:
            print("  roofline", {k: r.get(k) for k in ("bound", "kernel", "achieved", "peak", "frac")})
            sh = r.get("step_hbm") or {}
            print("  step_hbm single", sh.get("frac_single_pass"), "two", sh.get("frac_two_pass"),
                  "share", r.get("stage_share_of_step"))
        kk = d.get("kernels")
        if kk:
            print("  kernels", {k: (round(v["ms"], 4) if isinstance(v, dict) and "ms" in v else None)
                                for k, v in kk.items()},
                  "fp64", kk.get("search", {}).get("frac_fp64"),
                  "hist", kk.get("histogram", {}).get("frac_hbm"), "label", kk.get("label", {}).get("frac_hbm"))
        if d.get("e2e"):
            print("  e2e", d["e2e"].get("value"))
        c = d.get("cpu_baseline")
        if c:
            print("  cpu", c.get("value"), c.get("cores"), c.get("one_thread"), c.get("sample"))
        print("  clocks", d.get("clocks"), d.get("note"))
        if d.get("provenance"):
            print("  prov", d["provenance"])
