"""Per-slice phase timeline of k_scan_seed (debug build tools/build/libtsa_trace.so,
-DTSA_TRACE): start, histogram staged, tables (k_scan body), rows staged,
records + grid, grid reduce, ascent, end.  python tools/scan_trace.py [c5]"""
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
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = phantom.CONFIGS[name]
vol = torch.from_numpy(phantom.make_volume(cfg)).cuda()
for _ in range(3):
    tsa.tsa_segment(vol, cfg.bins, cfg.k, cfg.qs[0])
torch.cuda.synchronize()
lib.tsa_debug_mphase.argtypes = [ctypes.c_void_p, ctypes.c_int]
ph = np.zeros(8 * 4096, np.uint64)
lib.tsa_debug_mphase(ph.ctypes.data, cfg.nz)
ph = ph[: 8 * cfg.nz].reshape(cfg.nz, 8).astype(np.int64)
t0 = ph[:, 0].min()
d = np.diff(ph, axis=1) / 1e3
names = ["hist stage", "tables (k_scan body)", "rows stage", "records+grid", "grid reduce", "ascent", "end"]
print(f"{name}: kernel span {(ph[:, 7].max() - t0) / 1e3:.1f} us, CTA duration mean "
      f"{((ph[:, 7] - ph[:, 0]) / 1e3).mean():.1f} us")
print("  phases (mean us):", ", ".join(f"{n} {v:.2f}" for n, v in zip(names, d.mean(axis=0))))
st = (ph[:, 0] - t0) / 1e3
print("  CTA start times (us) percentiles 0/25/50/75/100:", np.percentile(st, [0, 25, 50, 75, 100]).round(1))

lib.tsa_debug_sphase.argtypes = [ctypes.c_void_p, ctypes.c_int]
sp = np.zeros(8 * 4096, np.uint64)
lib.tsa_debug_sphase(sp.ctypes.data, cfg.nz)
sp = sp[: 8 * cfg.nz].reshape(cfg.nz, 8).astype(np.int64)
d = np.diff(sp[:, :7], axis=1) / 1e3
names = ["pow (all bins, lane-strided)", "per-thread prefix", "block scan", "table writes", "status/M", "Asuf + rows"]
print("  table phases (mean us):", ", ".join(f"{n} {v:.2f}" for n, v in zip(names, d.mean(axis=0))))
