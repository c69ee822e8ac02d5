"""Quick CUDA-event timing of the 2-D path (tsa2d_segment) on the c2 phantom.

    python tools/time2d.py [--nz 300] [--cluster 0] [--reps 50] [--q 0.8] [--hist-only]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import phantom  # noqa: E402
import paper_2012_10684_b200 as tsa  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nz", type=int, default=300)
    ap.add_argument("--cluster", type=int, default=0)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--q", type=float, default=0.8)
    ap.add_argument("--hist-only", action="store_true")
    ap.add_argument("--no-labels", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    vol = torch.from_numpy(phantom.make_volume(phantom.CONFIGS["c2"], nz=a.nz)).to(dev)
    vols = [vol] + [vol.clone() for _ in range(3)]
    p = tsa.make_problem2d(vol, 256, a.q, a.cluster)
    ws = tsa.tsa2d_workspace(tsa.make_problem2d(vol, 256, 1.0 if a.hist_only else a.q, a.cluster), dev)
    print("cluster", tsa.tsa2d_cluster_size(vol, 256, a.q, a.cluster))

    def step(v):
        if a.hist_only:
            return tsa.tsa2d_histogram(v, 256, cluster=a.cluster, workspace=ws)
        return tsa.tsa2d_segment(v, 256, a.q, labels=not a.no_labels, cluster=a.cluster,
                                 workspace=ws)

    outs = [step(v) for v in vols]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.reps):
        step(vols[i % len(vols)])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"nz={a.nz} step {ms * 1e3:.1f} us  {a.nz / ms * 1e3:.0f} slices/s")
    if not a.hist_only:
        print("t,s of slices 0,150:", outs[0]["thresholds"][0].tolist(),
              outs[0]["thresholds"][min(150, a.nz - 1)].tolist())


if __name__ == "__main__":
    main()
