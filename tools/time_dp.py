"""CUDA-event timing: tsa_segment with the exact DP vs the exhaustive canonical
search on a BASELINE config (default c4: k = 4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import phantom  # noqa: E402
import paper_2012_10684_b200 as tsa  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = phantom.CONFIGS[name]
vol = torch.from_numpy(phantom.make_volume(cfg)).cuda()
for enum in ("dp", "canonical"):
    for q in cfg.qs[:1] + ((1.0, 1.4) if name == "c4" else ()):
        for _ in range(3):
            tsa.tsa_segment(vol, cfg.bins, cfg.k, q, enumeration=enum)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 20
        for _ in range(n):
            tsa.tsa_segment(vol, cfg.bins, cfg.k, q, enumeration=enum)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} k={cfg.k} q={q} {enum:9s} {e0.elapsed_time(e1) / n * 1e3:9.1f} us/step")
