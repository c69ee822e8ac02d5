"""PCIe experiment for the e2e path: raw pinned H2D / D2H rates and
tsa_segment_host with several slab sizes (c2)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import phantom  # noqa: E402
import paper_2012_10684_b200 as tsa  # noqa: E402

cfg = phantom.CONFIGS["c2"]
host = torch.from_numpy(phantom.make_volume(cfg)).pin_memory()
dev = torch.empty_like(host, device="cuda")
out = torch.empty_like(host).pin_memory()
for name, fn in (("H2D", lambda: dev.copy_(host, non_blocking=True)),
                 ("D2H", lambda: out.copy_(dev, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    print(f"{name} {host.nbytes / dt / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        dev.copy_(host, non_blocking=True)
    with torch.cuda.stream(s2):
        out.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 10
print(f"H2D || D2H {2 * host.nbytes / dt / 1e9:.1f} GB/s total")
for slab in (10, 25, 50, 75, 150):
    o = None
    for it in range(3):
        t = time.perf_counter()
        o = tsa.tsa_segment_host(host, 256, 2, 0.8, slab=slab, out=o)
        dt = time.perf_counter() - t
    print(f"slab {slab}: {cfg.nz / dt:.0f} slices/s ({dt * 1e3:.2f} ms)")

# decoupled pipeline emulation: H2D on a copy-in stream, compute on the compute
# stream, D2H on a copy-out stream, events between; NB buffers
import numpy as np  # noqa: E402

def pipelined(slab, nb):
    nz = cfg.nz
    sin, scomp, sout = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    dvol = [torch.empty((slab, cfg.ny, cfg.nx), dtype=torch.uint8, device="cuda") for _ in range(nb)]
    dlab = [torch.empty_like(d) for d in dvol]
    p = tsa.make_problem(dvol[0], 256, 2, 0.8)
    ws = [tsa.workspace_for(p, torch.device("cuda")) for _ in range(nb)]
    outs = [{"thresholds": torch.empty((slab, 2), dtype=torch.int32, device="cuda"),
             "objective": torch.empty(slab, dtype=torch.float64, device="cuda"),
             "histogram": None, "status": torch.empty(slab, dtype=torch.int32, device="cuda"),
             "labels": dlab[i]} for i in range(nb)]
    freed = [None] * nb
    t = time.perf_counter()
    for i, z0 in enumerate(range(0, nz, slab)):
        b = i % nb
        n = min(slab, nz - z0)
        if freed[b] is not None:
            sin.wait_event(freed[b])
        with torch.cuda.stream(sin):
            dvol[b][:n].copy_(host[z0:z0 + n], non_blocking=True)
            e_in = torch.cuda.Event()
            e_in.record(sin)
        scomp.wait_event(e_in)
        o = dict(outs[b])
        if n < slab:
            o = {k: (v[:n] if v is not None else None) for k, v in o.items()}
        tsa.tsa_segment(dvol[b][:n], 256, 2, 0.8, out=o, workspace=ws[b], stream=scomp)
        e_c = torch.cuda.Event()
        e_c.record(scomp)
        sout.wait_event(e_c)
        with torch.cuda.stream(sout):
            out[z0:z0 + n].copy_(dlab[b][:n], non_blocking=True)
            freed[b] = torch.cuda.Event()
            freed[b].record(sout)
    torch.cuda.synchronize()
    return time.perf_counter() - t

for slab in (10, 20, 30, 50):
    for nb in (2, 3, 4):
        pipelined(slab, nb)
        dt = min(pipelined(slab, nb) for _ in range(3))
        print(f"pipelined slab {slab} nb {nb}: {cfg.nz / dt:.0f} slices/s ({dt * 1e3:.2f} ms)")
