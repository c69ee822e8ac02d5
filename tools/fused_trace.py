"""Task-level timeline of the fused kernel (debug build tools/build/libtsa_trace.so,
compiled with -DTSA_TRACE).  Prints per-type busy time, waits and the timeline
span of each phase."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2012_10684_b200 as tsa
import phantom

tsa.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "build", "libtsa_trace.so")
lib = tsa.load()
lib.tsa_debug_trace.restype = ctypes.c_int
lib.tsa_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
pipe = sys.argv[2] if len(sys.argv) > 2 else "fused"
sb = int(sys.argv[3]) if len(sys.argv) > 3 else 16
dl = int(sys.argv[4]) if len(sys.argv) > 4 else 6
cfg = phantom.CONFIGS[name]
vol = torch.from_numpy(phantom.make_volume(cfg)).cuda()
for _ in range(3):
    tsa.tsa_segment(vol, cfg.bins, cfg.k, cfg.qs[0], pipeline=pipe, slab_slices=sb, label_lag=dl)
torch.cuda.synchronize()
buf = np.zeros(5 * 65536, np.uint64)
lib.tsa_debug_trace(buf.ctypes.data, 65536)  # reset
tsa.tsa_segment(vol, cfg.bins, cfg.k, cfg.qs[0], pipeline=pipe, slab_slices=sb, label_lag=dl)
torch.cuda.synchronize()
n = lib.tsa_debug_trace(buf.ctypes.data, 65536)
tr = buf[: 5 * n].reshape(n, 5).astype(np.int64)
t0 = tr[:, 3].min()
span = (tr[:, 4].max() - t0) / 1e3
print(f"{name} {pipe} sb={sb} dl={dl}: {n} tasks, kernel span {span:.1f} us")
for ty, nm in ((0, "LUT/noop"), (1, "H"), (2, "M"), (3, "L")):
    m = tr[:, 0] == ty
    if not m.any():
        continue
    d = (tr[m, 4] - tr[m, 3]) / 1e3
    print(f"  {nm:8s} n={m.sum():5d} mean {d.mean():7.2f} us  p50 {np.median(d):7.2f}  max {d.max():7.2f}  "
          f"sum {d.sum():9.1f} us  first start {(tr[m,3].min()-t0)/1e3:6.1f}  last end {(tr[m,4].max()-t0)/1e3:6.1f}")

lib.tsa_debug_mphase.argtypes = [ctypes.c_void_p, ctypes.c_int]
ph = np.zeros(8 * 4096, np.uint64)
lib.tsa_debug_mphase(ph.ctypes.data, cfg.nz)
ph = ph[: 8 * cfg.nz].reshape(cfg.nz, 8).astype(np.int64)
d = np.diff(ph[:, :7], axis=1) / 1e3
names = ["wait(LUT,H)", "hist+pow", "scan", "Asuf/Apre", "search+reduce", "finalize"]
print("  M phases (mean us):", ", ".join(f"{n} {v:.2f}" for n, v in zip(names, d.mean(axis=0))))
