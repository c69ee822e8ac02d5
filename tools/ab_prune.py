"""A/B of the bounded k = 2 search (TSA_K2_PRUNE=1, default) against the
plain exhaustive kernel (TSA_K2_PRUNE=0): whole tsa_segment step time on a
BASELINE config and bit-equality of every output.
python tools/ab_prune.py c5 [--reps 20] [--q 0.8]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import phantom  # noqa: E402
import paper_2012_10684_b200 as tsa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--q", type=float, default=None)
ap.add_argument("--pipeline", default="auto")
ap.add_argument("--var", default="TSA_K2_PRUNE", help="environment switch to A/B (0 = off, 1 = on)")
a = ap.parse_args()
cfg = phantom.CONFIGS[a.workload]
vol = torch.from_numpy(phantom.make_volume(cfg)).cuda()
q = cfg.qs[0] if a.q is None else a.q
p = tsa.make_problem(vol, cfg.bins, cfg.k, q, pipeline=a.pipeline)
ws = tsa.workspace_for(p, vol.device)
outs = {}
for flag in ("0", "1", "0", "1"):
    os.environ[a.var] = flag
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(a.reps):
        e0.record()
        out = tsa.tsa_segment(vol, cfg.bins, cfg.k, q, pipeline=a.pipeline, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{a.workload} q={q} {a.var}={flag} kind={tsa.tsa_pipeline_kind(p)} median {ts[len(ts)//2]:.4f} ms "
          f"min {ts[0]:.4f} ms", flush=True)
    outs[flag] = {k: v.clone() for k, v in out.items() if v is not None}
for k in outs["0"]:
    x, y = outs["0"][k], outs["1"][k]
    same = torch.equal(x.view(torch.int64) if x.dtype == torch.float64 else x,
                       y.view(torch.int64) if y.dtype == torch.float64 else y)
    print(f"  {k}: {'bit-identical' if same else 'DIFFERENT'}")
