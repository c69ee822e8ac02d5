"""Run tsa_segment on a BASELINE config a few times (for ncu / nsys-less
profiling): python tools/prof_run.py c5 [--pipeline stream|staged|auto] [--reps 3]
[--nz N] [--q Q]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import phantom  # noqa: E402
import paper_2012_10684_b200 as tsa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--pipeline", default="auto")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--nz", type=int, default=0)
ap.add_argument("--q", type=float, default=None)
ap.add_argument("--enumeration", default="canonical")
ap.add_argument("--hc", type=int, default=0)
ap.add_argument("--lag", type=int, default=0)
a = ap.parse_args()
cfg = phantom.CONFIGS[a.workload]
vol = torch.from_numpy(phantom.make_volume(cfg, nz=a.nz or None)).cuda()
q = cfg.qs[0] if a.q is None else a.q
p = tsa.make_problem(vol, cfg.bins, cfg.k, q, enumeration=a.enumeration, pipeline=a.pipeline,
                     slab_slices=a.hc, label_lag=a.lag)
ws = tsa.workspace_for(p, vol.device)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(a.reps):
    e0.record()
    tsa.tsa_segment(vol, cfg.bins, cfg.k, q, enumeration=a.enumeration, pipeline=a.pipeline, workspace=ws,
                    slab_slices=a.hc, label_lag=a.lag)
    e1.record()
    torch.cuda.synchronize()
    print(f"{a.workload} pipeline={a.pipeline} kind={tsa.tsa_pipeline_kind(p)} rep {i}: {e0.elapsed_time(e1):.3f} ms",
          flush=True)
