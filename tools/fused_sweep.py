"""Sweep the fused pipeline schedule (slab_slices x label_lag) on a workload."""
import statistics
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import phantom
import paper_2012_10684_b200 as tsa

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = phantom.CONFIGS[name]
host = phantom.make_volume(cfg)
vols = [torch.from_numpy(host).cuda() for _ in range(3)]
k, bins, q = cfg.k, cfg.bins, cfg.qs[0]
outs = [tsa.tsa_segment(v, bins, k, q) for v in vols]
ws = tsa.workspace_for(tsa.make_problem(vols[0], bins, k, q), "cuda")


def run(**kw):
    for i in range(10):
        tsa.tsa_segment(vols[i % 3], bins, k, q, out=outs[i % 3], workspace=ws, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 200
    for i in range(n):
        tsa.tsa_segment(vols[i % 3], bins, k, q, out=outs[i % 3], workspace=ws, **kw)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


print(f"{name} staged: {run(pipeline='staged'):.1f} us/step")
print(f"{name} compact: {run(pipeline='compact'):.1f} us/step")
for sb in (4, 8, 16, 32):
    for dl in (3, 4, 5, 6, 8, 12):
        print(f"{name} fused sb={sb} dl={dl}: {run(pipeline='fused', slab_slices=sb, label_lag=dl):.1f} us/step")
