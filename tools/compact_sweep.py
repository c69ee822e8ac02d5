"""Sweep compact-path knobs (hist CTAs per SM via slab_slices, k_mid threads via label_lag)."""
import os
import sys

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
    n = 300
    for i in range(n):
        tsa.tsa_segment(vols[i % 3], bins, k, q, out=outs[i % 3], workspace=ws, **kw)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for hs in (2, 3, 4):
    for mt in (256,):
        print(f"{name} compact hist_ctas_per_sm={hs or 'auto'} mid_threads={mt}: "
              f"{run(pipeline='compact', slab_slices=hs, label_lag=mt):.1f} us/step", flush=True)
