#!/usr/bin/env python
"""Benchmark of the Tsallis multilevel-thresholding hot path (arXiv 2012.10684).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl reference]

(--workload f1: the paper's own 2-D formulation, on the
c2 volume; tsa2d_segment per step.)

A *step* is one pass of the whole hot path (SURVEY.md §8(a) rows a1-a5:
histogram -> prefix tables -> exhaustive tuple search -> argmax/finalize ->
labels) over one synthetic CT volume of the workload (default c2 =
BASELINE.json:configs[1], 512x512x300 u8, 256 bins, k=2, q=0.8).  With N GPUs
(torchrun, one process per GPU) every rank segments its own resident volume
(slices sharded over GPUs, no data-path collective): weak scaling,
value = slices of all ranks / max-over-ranks device time.

Prints ONE JSON line on rank 0 (metric, value, unit, ..., roofline,
cpu_baseline, e2e, clocks, gpu_launches).  --impl reference times the CPU
oracle (the reference arm for this paper, which has no code of its own).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CT slices/sec and Gtuples/s Tsallis search at 1/2/4/8 B200 vs roofline"
UNIT = "slices/s"
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, only if MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c5",
                    help="c1..c5 (BASELINE.json configs; default c5, the largest single-GPU config), "
                         "f1 (2-D), f2 (HU input), f3 (morphology)")
    ap.add_argument("--dry-run", action="store_true", help="launcher check only (no GPU work)")
    ap.add_argument("--impl", default="tsa", choices=["tsa", "reference"])
    ap.add_argument("--enumeration", default="canonical", choices=["canonical", "full", "dp"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-slab", type=int, default=0, help="slices per host<->device slab (0 = default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--buffers", type=int, default=0, help="resident volume copies rotated (0 = auto, > 2x L2)")
    ap.add_argument("--shard", default="auto", choices=["auto", "slabs", "replicas", "tuples"],
                    help="slabs: one volume split into per-rank slabs, no collective (strong scaling; "
                         "default); replicas: every rank its own volume (weak); tuples: the ranks split "
                         "the tuple space of every slice, NCCL all-gathers inside libtsa (default for c4)")
    ap.add_argument("--pipeline", default="auto", choices=["auto", "compact", "fused", "staged"])
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": HBM_FALLBACK_GBS}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms in the background."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append((time.perf_counter(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        win = [p for (t, p) in self.samples if t0 - 0.05 <= t <= t1 + 0.05]
        if len(win) < 3:  # timed region shorter than the sampling period: widen
            win = [p for (t, p) in self.samples if t0 - 2.0 <= t <= t1 + 0.5]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(p[0]) for p in win if p[0].replace(".", "").isdigit()]
        mx = [float(p[1]) for p in win if p[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for p in win for n, v in zip(names, p[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(win)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(x, world, device):
    import torch

    if world == 1:
        return x
    import torch.distributed as dist

    gloo = dist.get_backend() == "gloo"
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if gloo else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def cpu_baseline(cfg, vol, qs, target_s=10.0):
    """The oracle as it stands, on the host cores, over a bounded sample of the
    workload: whole-volume passes (or a slice prefix) repeated until about
    target_s seconds of wall time (capped at 20 passes); every q of the
    workload per pass (c3: the 11-q sweep, histogram and labels included each
    time, as the oracle has no sweep).  Also one slice on one thread
    (extrapolated per-core rate)."""
    import oracle

    qs = tuple(qs) if isinstance(qs, (tuple, list)) else (qs,)
    threads = oracle.max_threads()

    def run(n, th=threads):
        for q in qs:
            oracle.segment(vol[:n], cfg.bins, cfg.k, q, threads=th)

    n0 = min(cfg.nz, max(threads, 4))
    t = time.perf_counter()
    run(n0)
    dt = time.perf_counter() - t
    n = int(min(cfg.nz, max(n0, n0 * target_s / max(dt, 1e-6))))
    reps, slices, t = 0, 0, time.perf_counter()
    while True:
        run(n)
        reps += 1
        slices += n
        el = time.perf_counter() - t
        if el >= target_s or reps >= 20:
            break
    z1 = cfg.nz // 2
    t = time.perf_counter()
    for q in qs:
        oracle.segment(vol[z1:z1 + 1], cfg.bins, cfg.k, q, threads=1)
    one = time.perf_counter() - t
    return {"value": slices / el, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{reps} pass(es) over the first {n} of {cfg.nz} slices of workload {cfg.name} "
                      f"(whole path: histogram, exhaustive Level-1 search, labels"
                      f"{', all ' + str(len(qs)) + ' q' if len(qs) > 1 else ''}), {threads} OpenMP threads, "
                      f"{el:.2f} s",
            "one_thread": {"slices_per_s": 1.0 / one, "sample": f"slice {z1}, 1 thread, {one:.2f} s",
                           "extrapolated_full_volume_s": one * cfg.nz}}


def run_reference(args, cfg, rank, world):
    """Reference arm: the CPU oracle, timed as it stands (rank 0 only)."""
    import numpy as np

    import oracle
    import phantom

    if rank != 0:
        return
    if cfg.name == "f1":
        run_reference_2d(args, cfg, world)
        return
    vol = phantom.make_volume(cfg)
    threads = oracle.max_threads()
    qs = cfg.qs if cfg.name in ("c1", "c2", "c3", "c4", "c5") else cfg.qs[:1]
    if cfg.name == "f2":  # HU input: the pre-processing oracle, then the 1-D oracle
        def seg(v, threads=None):
            g, _, _ = oracle.preprocess(v)
            return oracle.segment(g, 256, cfg.k, qs[0], threads=threads)
        what = "pre-processing + whole 1-D path"
    elif cfg.name == "f3":  # disk(10) top-hat, brute force
        def seg(v, threads=None):
            return oracle.tophat(v, cfg.k)
        what = f"brute-force disk({cfg.k}) opening + top-hat, single-threaded"
    else:
        def seg(v, threads=None):
            for q in qs:
                oracle.segment(v, cfg.bins, cfg.k, q, threads=threads)
        what = "whole path, Level-1 oracle" + (f", all {len(qs)} q per slice" if len(qs) > 1 else "")
    # a step = spp slices (a multiple of the thread count when a slice is slow),
    # sized so warm-up + timed steps take about `budget` seconds; if even one
    # such step per requested step exceeds it, fewer steps are timed (stated).
    t = time.perf_counter()
    seg(vol[:threads], threads=threads)
    per_batch = time.perf_counter() - t  # `threads` slices in parallel
    per_slice = per_batch / threads
    budget = 150.0
    nsteps = max(args.steps + args.warmup, 1)
    spp = int(max(1, min(cfg.nz, budget / nsteps / max(per_slice, 1e-6))))
    if spp < threads and per_batch * nsteps > budget:
        spp = min(cfg.nz, threads)  # one parallel batch per step; time fewer steps
    per_step = per_batch * max(1, spp / threads)
    timed = int(max(1, min(args.steps, (budget - min(args.warmup, 1) * per_step) / max(per_step, 1e-6))))
    warm = min(args.warmup, 1 if timed < args.steps else args.warmup)
    for _ in range(warm):
        seg(vol[:spp], threads=threads)
    t = time.perf_counter()
    for s_ in range(timed):
        z0 = (s_ * spp) % max(1, cfg.nz - spp + 1)
        seg(vol[z0:z0 + spp], threads=threads)
    dt = time.perf_counter() - t
    value = spp * timed / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / timed,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_for(cfg, args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{spp} slices of {cfg.name} per step ({what})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if timed < args.steps:
        line["steps_timed"] = timed
        line["note"] = (f"{timed} of the {args.steps} requested steps timed (each {per_step:.1f} s of "
                        f"oracle work) to keep the run within about {budget:.0f} s; warm-up {warm}")
    print(json.dumps(line), flush=True)


def run_reference_2d(args, cfg, world):
    """Reference arm of the 2-D workload: oracle.segment2d (Level-0 exhaustive
    (t,s) search on all host cores) over a bounded slice sample per step."""
    import oracle
    import phantom

    q = cfg.qs[0]
    threads = oracle.max_threads()
    t = time.perf_counter()
    vol = phantom.make_volume(cfg, nz=8, z_first=100)
    oracle.segment2d(vol, cfg.bins, q, z_list=[0], threads=threads)
    per_slice = time.perf_counter() - t
    spp = max(1, int(min(8, 150.0 / max(args.steps + args.warmup, 1) / max(per_slice, 1e-6))))
    for _ in range(args.warmup):
        oracle.segment2d(vol, cfg.bins, q, z_list=range(spp), threads=threads)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle.segment2d(vol, cfg.bins, q, z_list=range(spp), threads=threads)
    dt = time.perf_counter() - t
    value = spp * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_of_2d(cfg, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{spp} slices of f1 per step (mean image, 2-D histogram, Level-0 "
                                   f"exhaustive (t,s) search, labels)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_of_2d(cfg, world):
    return {"workload": f"{cfg.name}: {cfg.note}", "nx": cfg.nx, "ny": cfg.ny,
            "slices_per_gpu": cfg.nz, "bins": cfg.bins, "q": cfg.qs[0], "input": cfg.dtype,
            "method": "2-D Tsallis: 3x3 mean image, L x L histogram, exhaustive (t,s), labels [f > t]",
            "parallelism": f"slices sharded, {world} GPU(s), no collective",
            "l2": "inputs larger than L2: rotating resident volume/label copies (> 2x 126 MB)"}


def run_2d(args, cfg, rank, world, dev):
    """The 2-D workload: a step = tsa2d_segment of the
    whole resident volume (k2d_luts + k_tsallis2d cluster kernel + labels)."""
    import numpy as np
    import torch

    import phantom
    import paper_2012_10684_b200 as tsa

    q, L = cfg.qs[0], cfg.bins
    host = phantom.make_volume(cfg)
    n_vox = host.size
    nbuf = args.buffers or max(2, int(np.ceil(2 * 126e6 / (2 * n_vox))) + 1)
    vols = [torch.from_numpy(host).to(dev) for _ in range(nbuf)]
    p = tsa.make_problem2d(vols[0], L, q)
    ws = tsa.tsa2d_workspace(p, dev)
    outs = [{"thresholds": torch.empty((cfg.nz, 2), dtype=torch.int32, device=dev),
             "objective": torch.empty(cfg.nz, dtype=torch.float64, device=dev),
             "status": torch.empty(cfg.nz, dtype=torch.int32, device=dev),
             "labels": torch.empty(host.shape, dtype=torch.uint8, device=dev),
             "histogram": None} for _ in range(nbuf)]
    stream = torch.cuda.current_stream()

    def step(i, labels=True):
        o = outs[i % nbuf] if labels else dict(outs[i % nbuf], labels=None)
        tsa.tsa2d_segment(vols[i % nbuf], L, q, out=o, workspace=ws, stream=stream)

    sampler = ClockSampler(dev.index)
    sampler.start()
    for i in range(max(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.perf_counter()
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    barrier(world)
    ms_per_step = max_over_ranks(e0.elapsed_time(e1), world, dev) / args.steps
    value = world * cfg.nz / (ms_per_step * 1e-3)

    # kernel split: luts + cluster kernel (no labels) vs labels alone
    reps = max(20, min(args.steps, 200))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    tcol = [o["thresholds"][:, :1].contiguous() for o in outs]
    for i in range(reps + 3):
        j = i - 3
        if j >= 0:
            ev[j][0].record(stream)
        step(i, labels=False)
        if j >= 0:
            ev[j][1].record(stream)
        tsa.tsa_label(vols[i % nbuf], tcol[i % nbuf], outs[i % nbuf]["status"], bins=L)
        if j >= 0:
            ev[j][2].record(stream)
    torch.cuda.synchronize()
    ms_main = statistics.mean(a.elapsed_time(b) for a, b, _ in ev)
    ms_lab = statistics.mean(b.elapsed_time(c) for _, b, c in ev)
    pk_, how = peaks()
    hbm = float(pk_.get("hbm_gbs", HBM_FALLBACK_GBS))
    main_bytes = n_vox  # the cluster kernel reads every pixel once (halo rows from L2)
    step_bytes = 2 * n_vox  # volume once + labels once
    kernels = {
        "k_tsallis2d": {"ms": ms_main, "bytes": main_bytes, "gbs": main_bytes / (ms_main * 1e-3) / 1e9,
                        "note": "k2d_luts + k_tsallis2d (histogram, walks, argmax); candidates "
                                f"{cfg.nz * (L - 1) ** 2} nominal"},
        "label": {"ms": ms_lab, "bytes": 2 * n_vox, "gbs": 2 * n_vox / (ms_lab * 1e-3) / 1e9},
        "cluster": tsa.tsa2d_cluster_size(vols[0], L, q),
    }
    tr = {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f).get(args.workload, {})
    roofline = {"bound": "hbm", "kernel": "k_tsallis2d (+ k2d_luts)",
                "achieved": kernels["k_tsallis2d"]["gbs"], "peak": hbm, "unit": "GB/s",
                "frac": kernels["k_tsallis2d"]["gbs"] / hbm, "traffic": tr.get("k_tsallis2d"),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({how})",
                "algorithmic_bytes_per_launch": main_bytes,
                "note": "on-chip bound (shared-memory atomics, latency of the summed-area walks); "
                        "the HBM fraction is the honest distance to the streaming floor"}

    # e2e through the public API: pinned H2D, tsa2d_segment, D2H of every output
    host_t = torch.from_numpy(host).pin_memory()
    hout = {"thresholds": torch.empty((cfg.nz, 2), dtype=torch.int32).pin_memory(),
            "objective": torch.empty(cfg.nz, dtype=torch.float64).pin_memory(),
            "status": torch.empty(cfg.nz, dtype=torch.int32).pin_memory(),
            "labels": torch.empty(host.shape, dtype=torch.uint8).pin_memory()}
    dvol = torch.empty_like(vols[0])

    def e2e_step():
        dvol.copy_(host_t, non_blocking=True)
        o = tsa.tsa2d_segment(dvol, L, q, out=outs[0], workspace=ws, stream=stream)
        for kk in hout:
            hout[kk].copy_(o[kk], non_blocking=True)
        torch.cuda.synchronize()

    e2e = None
    if args.e2e_steps > 0:
        e2e_step()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        dt = max_over_ranks(time.perf_counter() - t0, world, dev)
        e2e = {"value": world * cfg.nz * args.e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(host.nbytes),
               "d2h_bytes_per_step": int(sum(t.numel() * t.element_size() for t in hout.values())),
               "api": "pinned H2D copy + tsa2d_segment + D2H of thresholds/objective/status/labels",
               "steps": args.e2e_steps}
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        threads = oracle.max_threads()
        n, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < 10.0 and n < cfg.nz:
            oracle.segment2d(host[n:n + 1], L, q, threads=threads)
            n += 1
        el = time.perf_counter() - t0
        cpu = {"value": n / el, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"the first {n} of {cfg.nz} slices of f1 (mean image, 2-D histogram, Level-0 "
                         f"exhaustive (t,s) search, labels), {threads} OpenMP threads, {el:.1f} s"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of_2d(cfg, world), "roofline": roofline, "cpu_baseline": cpu,
            "e2e": e2e, "clocks": clocks, "gpu_launches": 3 * args.steps, "kernels": kernels,
            "pipeline": "2d-cluster",
            "gcandidates_per_s_nominal": world * cfg.nz * (L - 1) ** 2 / (ms_per_step * 1e-3) / 1e9,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_hu(args, cfg, rank, world, dev):
    """The HU workload: a step = tsa_hu_segment of the
    resident int16 volume (HU histograms + window, 8-bit remap, search,
    finalize, labels from HU)."""
    import numpy as np
    import torch

    import phantom
    import paper_2012_10684_b200 as tsa

    q, k = cfg.qs[0], cfg.k
    host = phantom.make_volume(cfg)
    n_vox = host.size
    nbuf = args.buffers or max(2, int(np.ceil(2 * 126e6 / (3 * n_vox))) + 1)
    vols = [torch.from_numpy(host).to(dev) for _ in range(nbuf)]
    p = tsa.make_hu_problem(vols[0], k, q)
    ws = tsa.tsa_hu_workspace(p, dev)
    outs = [{"thresholds": torch.empty((cfg.nz, k), dtype=torch.int32, device=dev),
             "objective": torch.empty(cfg.nz, dtype=torch.float64, device=dev),
             "histogram": torch.empty((cfg.nz, 256), dtype=torch.int32, device=dev),
             "status": torch.empty(cfg.nz, dtype=torch.int32, device=dev),
             "labels": torch.empty(host.shape, dtype=torch.uint8, device=dev),
             "window": torch.empty(2, dtype=torch.int32, device=dev)} for _ in range(nbuf)]
    stream = torch.cuda.current_stream()

    def step(i):
        tsa.tsa_hu_segment(vols[i % nbuf], k, q, out=outs[i % nbuf], workspace=ws, stream=stream)

    sampler = ClockSampler(dev.index)
    sampler.start()
    for i in range(max(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.perf_counter()
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    barrier(world)
    ms_per_step = max_over_ranks(e0.elapsed_time(e1), world, dev) / args.steps
    value = world * cfg.nz / (ms_per_step * 1e-3)
    pk_, how = peaks()
    hbm = float(pk_.get("hbm_gbs", HBM_FALLBACK_GBS))
    # algorithmic bytes of the step: the HU volume twice (histogram/window pass,
    # label pass) + the labels once
    step_bytes = 2 * 2 * n_vox + n_vox
    roofline = {"bound": "hbm", "kernel": "HU step (k_hu_hist + k_hu_remap + search + k_label_hu)",
                "achieved": step_bytes / (ms_per_step * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / hbm, "traffic": None,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({how})",
                "algorithmic_bytes_per_launch": step_bytes}
    host_t = torch.from_numpy(host).pin_memory()
    hout = {kk: torch.empty(v.shape, dtype=v.dtype).pin_memory() for kk, v in outs[0].items()}
    dvol = torch.empty_like(vols[0])

    def e2e_step():
        dvol.copy_(host_t, non_blocking=True)
        o = tsa.tsa_hu_segment(dvol, k, q, out=outs[0], workspace=ws, stream=stream)
        for kk in hout:
            hout[kk].copy_(o[kk], non_blocking=True)
        torch.cuda.synchronize()

    e2e = None
    if args.e2e_steps > 0:
        e2e_step()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        dt = max_over_ranks(time.perf_counter() - t0, world, dev)
        e2e = {"value": world * cfg.nz * args.e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(host.nbytes),
               "d2h_bytes_per_step": int(sum(t.numel() * t.element_size() for t in hout.values())),
               "api": "pinned H2D copy + tsa_hu_segment + D2H of every output", "steps": args.e2e_steps}
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        threads = oracle.max_threads()
        t0 = time.perf_counter()
        n, reps = cfg.nz, 0
        while True:
            gray, _, _ = oracle.preprocess(host[:n])
            oracle.segment(gray, 256, k, q, threads=threads)
            reps += 1
            el = time.perf_counter() - t0
            if el >= 10.0 or reps >= 20:
                break
        cpu = {"value": reps * n / el, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"{reps} pass(es) over all {n} slices of f2 (oracle.preprocess "
                         f"single-threaded, then the Level-1 oracle on {threads} threads), {el:.1f} s"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_for(cfg, args, world),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            # k_hu_init, k_hu_hist, k_hu_window, k_hu_window_fold, k_hu_glut,
            # k_hu_remap, k_lut_part, k_mid (per-slice search), k_label_hu
            "gpu_launches": (9 if cfg.k <= 2 else 11) * args.steps,
            "pipeline": "hu-fused (per-slice search kernel)" if cfg.k <= 2 else "hu-fused (staged search)",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def morph_roofline(r, n_vox, ms_per_step, clocks, dev):
    """ALU roofline of the top-hat step: per pixel and pass the
    exact disk erosion/dilation needs r + 1 min/max ops for the horizontal
    running extrema H_1..H_r and 2r for the fold over the 2r + 1 disk rows;
    the top-hat adds a max and a subtraction: 6r + 4 byte ops per pixel.  Peak:
    the ALU pipe issues 16 lanes/clk per SMSP (B300_MICROARCH.md "Pipe rates":
    rt_SMSP = 2), 4 SMSPs per SM, 2 byte ops per VIMNMX.U16x2 / VIADD.16x2
    lane, at the SM clock sampled during the timed region."""
    import torch

    ops = (6 * r + 4) * n_vox
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = clocks.get("sm_max_mhz") or clocks.get("sm_mhz") or 1965.0
    peak = sms * 4 * 16 * 2 * mhz * 1e6 / 1e12
    achieved = ops / (ms_per_step * 1e-3) / 1e12
    pk_, how = peaks()
    hbm = float(pk_.get("hbm_gbs", HBM_FALLBACK_GBS))
    alg_bytes = 2 * n_vox  # the volume once + the mask once
    return {"bound": "alu", "kernel": "k_morph erode pass + k_morph dilate/top-hat pass",
            "achieved": achieved, "peak": peak, "unit": "Tops/s", "frac": achieved / peak,
            "traffic": None,
            "peak_source": f"derived: {sms} SMs x 4 SMSP x 16 ALU lanes/clk x 2 byte ops (16x2 SIMD) "
                           f"x {mhz:.0f} MHz (sm_max_mhz sampled in the timed region)",
            "algorithmic_ops_per_launch": ops, "ops_per_pixel": 6 * r + 4,
            "hbm": {"achieved_gbs": alg_bytes / (ms_per_step * 1e-3) / 1e9, "peak_gbs": hbm,
                    "frac": alg_bytes / (ms_per_step * 1e-3) / 1e9 / hbm,
                    "algorithmic_bytes_per_launch": alg_bytes,
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({how})"}}


def run_morph(args, cfg, rank, world, dev):
    """The morphology workload: a step = tsa_morph
    'tophat' with disk(10) of the resident volume (erode pass + dilate pass
    with the fused subtraction)."""
    import numpy as np
    import torch

    import phantom
    import paper_2012_10684_b200 as tsa

    r = cfg.k
    host = phantom.make_volume(cfg)
    n_vox = host.size
    nbuf = args.buffers or max(2, int(np.ceil(2 * 126e6 / (2 * n_vox))) + 1)
    vols = [torch.from_numpy(host).to(dev) for _ in range(nbuf)]
    outs = [torch.empty_like(vols[0]) for _ in range(nbuf)]
    ws = torch.empty(int(tsa.load().tsa_morph_workspace_size(cfg.nx, cfg.ny, cfg.nz, 3)),
                     dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(i):
        tsa.tsa_morph(vols[i % nbuf], "tophat", r, out=outs[i % nbuf], workspace=ws, stream=stream)

    sampler = ClockSampler(dev.index)
    sampler.start()
    for i in range(max(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.perf_counter()
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    barrier(world)
    ms_per_step = max_over_ranks(e0.elapsed_time(e1), world, dev) / args.steps
    value = world * cfg.nz / (ms_per_step * 1e-3)
    host_t = torch.from_numpy(host).pin_memory()
    hout = torch.empty(host.shape, dtype=torch.uint8).pin_memory()
    dvol = torch.empty_like(vols[0])

    def e2e_step():
        dvol.copy_(host_t, non_blocking=True)
        tsa.tsa_morph(dvol, "tophat", r, out=outs[0], workspace=ws, stream=stream)
        hout.copy_(outs[0], non_blocking=True)
        torch.cuda.synchronize()

    e2e = None
    if args.e2e_steps > 0:
        e2e_step()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        dt = max_over_ranks(time.perf_counter() - t0, world, dev)
        e2e = {"value": world * cfg.nz * args.e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(host.nbytes), "d2h_bytes_per_step": int(hout.nbytes),
               "api": "pinned H2D copy + tsa_morph(tophat) + D2H of the mask", "steps": args.e2e_steps}
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)
    roofline = morph_roofline(r, n_vox, ms_per_step, clocks, dev)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        n, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < 10.0 and n < cfg.nz:
            oracle.tophat(host[n], r)
            n += 1
        el = time.perf_counter() - t0
        cpu = {"value": n / el, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"the first {n} of {cfg.nz} slices of f3 (brute-force disk({r}) erosion, "
                         f"dilation, subtraction; single-threaded), {el:.1f} s"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": config_for(cfg, args, world),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": 2 * args.steps, "pipeline": "morph (2 streaming passes)",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def config_for(cfg, args, world):
    """The workload's config dict, identical in the GPU arm and the reference arm."""
    if cfg.name == "f1":
        return config_of_2d(cfg, world)
    if cfg.name == "f2":
        return dict(config_of(cfg, args, world), input="i16 HU (background -2000)")
    if cfg.name == "f3":
        return {"workload": f"{cfg.name}: {cfg.note}", "nx": cfg.nx, "ny": cfg.ny,
                "slices_per_gpu": cfg.nz, "radius": cfg.k, "op": "white top-hat = in - open(in)",
                "parallelism": f"slices sharded, {world} GPU(s), no collective",
                "l2": "inputs larger than L2: rotating resident volume copies"}
    return config_of(cfg, args, world)


def shard_mode(args, cfg, world):
    """slabs: one volume, rank r segments slices tsa_slab_range(nz, P, r), no
    collective (strong scaling); replicas: every rank its own
    full volume (weak); tuples: the tuple space of every slice split over the
    ranks, NCCL inside libtsa (c4's mode)."""
    if args.shard != "auto":
        return args.shard
    if cfg.name == "c4" and world > 1:
        return "tuples"
    return "slabs"


def config_of(cfg, args, world):
    mode = shard_mode(args, cfg, world)
    par = {"slabs": f"slices sharded: one {cfg.nz}-slice volume split into {world} contiguous slab(s) "
                    f"of <= {-(-cfg.nz // world)} slices, no collective",
           "replicas": f"{world} GPU(s), each segments its own {cfg.nz}-slice volume, no collective",
           "tuples": f"tuple space of every slice split over {world} GPU(s); histogram and (score, key) "
                     f"all-gathers over NCCL inside libtsa (tsa_segment_sharded)"}[mode]
    d = {"workload": f"{cfg.name}: {cfg.note}", "nx": cfg.nx, "ny": cfg.ny, "nz": cfg.nz,
         "bins": cfg.bins, "k": cfg.k, "q": list(cfg.qs) if len(cfg.qs) > 1 else cfg.qs[0],
         "input": cfg.dtype, "objective": "pseudo_additive", "enumeration": args.enumeration,
         "shard": mode, "parallelism": par,
         "l2": "inputs larger than L2: rotating resident volume/label copies (> 2x 126 MB)"}
    if len(cfg.qs) > 1:
        d["step"] = f"one histogram + search/finalize/labels for each of the {len(cfg.qs)} q (tsa_segment_sweep)"
    return d


def provenance(cfg, host, dev):
    """Run provenance: seed, volume SHA-256, host CPU, GPU, driver."""
    import hashlib

    import torch

    import phantom

    cpu = "?"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    drv = None
    try:
        drv = subprocess.check_output(["nvidia-smi", "--query-gpu=driver_version", "--format=csv,noheader",
                                       "-i", str(dev.index)], text=True, timeout=20).strip()
    except Exception:
        pass
    lib = os.path.join(ROOT, "paper_2012_10684_b200", "libtsa.so")
    with open(lib, "rb") as f:
        libsha = hashlib.sha256(f.read()).hexdigest()
    return {"seed": cfg.seed, "volume_sha256": phantom.sha256(host), "volume_shape": list(host.shape),
            "cpu_model": cpu, "host_cores": os.cpu_count(), "gpu": torch.cuda.get_device_name(dev),
            "sms": torch.cuda.get_device_properties(dev).multi_processor_count, "driver": drv,
            "cuda_runtime": torch.version.cuda, "torch": torch.__version__, "libtsa_sha256": libsha}


def fp64_peak():
    """Measured FP64 lane-op rate (tools/fp64_peak.cu, profiles/fp64_peak.json:
    DMUL lane-ops/s); else 148 SMs x 64 lanes x 1.965 GHz."""
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["dmul_lane_ops_per_s"]), "measured: profiles/fp64_peak.json dmul_lane_ops_per_s " \
                                                 "(tools/fp64_peak.cu DMUL chains, 148 SMs, 1965 MHz)"
    return 148 * 64 * 1.965e9, "nominal 148 SMs x 64 FP64 lanes x 1.965 GHz"


def fp64_per_tuple(k, q, enumeration):
    """Algorithmic FP64-pipe instructions per evaluated tuple.
    k >= 3: the prefix x suffix factorisation leaves 1 DMUL + 1 DSETP per tuple
    (SURVEY.md §8(d)).  k = 2: every tuple owns its middle class, whose term
    W / n^q is one expression tree: dd difference of W (3 DADD), d = r (1/j)
    2^-s (1 DMUL), j^-q 2^(-sq) (1 DMUL), the degree-DEG Horner polynomial
    (DEG DFMA), their product (1 DMUL), W n^-q (1 DMUL), the two combines
    (2 DMUL) and the compare (1 DSETP): 10 + DEG (DEG = 5 for q <= 2).  q == 1
    (Shannon) is counted the same way.  k = 1: one class term (as k = 2)."""
    if enumeration == "dp":
        return None
    if k >= 3:
        return 2
    deg = 5 if q <= 2 else (6 if q <= 10 else 12)
    return 10 + deg


def graph_time(fn, reps=10, replays=5):
    """Mean time of one fn() call: fn captured `reps` times in a CUDA graph,
    replayed `replays` times after one warm-up replay (device time, CUDA events
    on the replay stream; no host work or allocation inside)."""
    import torch

    s = torch.cuda.Stream()
    fn()  # warm (attribute calls, lazy loading) outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(replays):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * replays)


def stage_times(cfg, args, vols, nbuf, dev):
    """Per-stage device times from isolated launches (each stage captured in a
    CUDA graph with preallocated buffers, no allocation in the timed region).
    Returns ms per call of histogram, search (k_small_luts + k_scan [+ k_rtable]
    + search kernel + merge), finalize, label, for q = qs[0] (c3: every q)."""
    import torch

    import paper_2012_10684_b200 as tsa

    nz, bins, k = cfg.nz, cfg.bins, cfg.k
    N = cfg.nx * cfg.ny
    U = tsa.tsa_default_units(nz, bins, k, args.enumeration)
    hist = [torch.empty((nz, bins), dtype=torch.int32, device=dev) for _ in range(nbuf)]
    st = [torch.empty(nz, dtype=torch.int32, device=dev) for _ in range(nbuf)]
    st2 = [torch.empty(nz, dtype=torch.int32, device=dev) for _ in range(nbuf)]
    ps = torch.empty((U, nz), dtype=torch.float64, device=dev)
    pk = torch.empty((U, nz), dtype=torch.int64, device=dev)
    thr = torch.empty((nz, k), dtype=torch.int32, device=dev)
    phi = torch.empty(nz, dtype=torch.float64, device=dev)
    stf = torch.empty(nz, dtype=torch.int32, device=dev)
    lab = [torch.empty(vols[0].shape, dtype=torch.uint8, device=dev) for _ in range(nbuf)]
    wsb = max(tsa.tsa_search_workspace_size(nz, N, bins, k, q, 0, args.enumeration) for q in cfg.qs)
    sws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    for b in range(nbuf):
        tsa.tsa_histogram(vols[b], bins, out=(hist[b], st[b]))
    torch.cuda.synchronize()
    out = {"histogram": graph_time(lambda i=0: tsa.tsa_histogram(vols[i % nbuf], bins,
                                                                  out=(hist[i % nbuf], st[i % nbuf])))}
    per_q = []
    for q in cfg.qs:
        def search(i=0):
            st2[i % nbuf].copy_(st[i % nbuf])
            tsa.tsa_search(hist[i % nbuf], st2[i % nbuf], N, k, q, enumeration=args.enumeration, units=U,
                           workspace=sws, out=(ps, pk))

        def copy(i=0):
            st2[i % nbuf].copy_(st[i % nbuf])

        t_search = graph_time(search, reps=6, replays=3) - graph_time(copy)
        search()
        torch.cuda.synchronize()
        t_fin = graph_time(lambda i=0: tsa.tsa_finalize(hist[0], st2[0], k, q, ps, pk, out=(thr, phi, stf)))
        t_lab = graph_time(lambda i=0: tsa.tsa_label(vols[i % nbuf], thr, stf, bins=bins, out=lab[i % nbuf]))
        per_q.append({"q": q, "search": t_search, "finalize": t_fin, "label": t_lab})
    out["per_q"] = per_q
    for key in ("search", "finalize", "label"):
        out[key] = sum(d[key] for d in per_q)
    return out


def run_1d(args, cfg, rank, world, dev):
    """The 1-D path (BASELINE.json configs c1-c5): a step = tsa_segment of the
    rank's resident volume or slab (c3: tsa_segment_sweep over the 11 q)."""
    import ctypes
    from math import comb

    import numpy as np
    import torch

    import phantom
    import paper_2012_10684_b200 as tsa

    mode = shard_mode(args, cfg, world)
    k, bins, qs = cfg.k, cfg.bins, cfg.qs
    sweep = len(qs) > 1
    if mode == "slabs":
        z0, z1 = tsa.tsa_slab_range(cfg.nz, world, rank)
    else:
        z0, z1 = 0, cfg.nz
    host = phantom.make_volume(cfg, nz=z1 - z0, z_first=z0) if z1 > z0 else \
        np.zeros((0, cfg.ny, cfg.nx), cfg.np_dtype)
    nzl = host.shape[0]
    n_vox = host.size
    # resident copies so that consecutive steps never hit L2 (126 MB)
    nbuf = args.buffers or max(2, int(np.ceil(2 * 126e6 / max(host.nbytes + n_vox, 1))) + 1)
    vols = [torch.from_numpy(host).to(dev) for _ in range(nbuf)]
    outs, wss = [], None
    if nzl > 0:
        p = tsa.make_problem(vols[0], bins, k, qs[0], enumeration=args.enumeration, pipeline=args.pipeline)
        wss = tsa.sweep_workspace(vols[0], bins, k, qs, enumeration=args.enumeration) if sweep else \
            tsa.workspace_for(p, dev)
        for i in range(nbuf):
            hist_i = torch.empty((nzl, bins), dtype=torch.int32, device=dev)
            outs.append([{"thresholds": torch.empty((nzl, k), dtype=torch.int32, device=dev),
                          "objective": torch.empty(nzl, dtype=torch.float64, device=dev),
                          "histogram": hist_i if j == 0 else None,
                          "status": torch.empty(nzl, dtype=torch.int32, device=dev),
                          "labels": torch.empty(host.shape, dtype=torch.uint8, device=dev)}
                         for j in range(len(qs))])
    stream = torch.cuda.current_stream()

    def step(i):
        if nzl == 0:
            return
        o = outs[i % nbuf]
        if sweep:
            tsa.tsa_segment_sweep(vols[i % nbuf], bins, k, qs, enumeration=args.enumeration, outs=o,
                                  workspace=wss, stream=stream)
        else:
            tsa.tsa_segment(vols[i % nbuf], bins, k, qs[0], enumeration=args.enumeration, out=o[0],
                            workspace=wss, stream=stream, pipeline=args.pipeline)

    sampler = ClockSampler(dev.index)
    sampler.start()
    for i in range(max(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.perf_counter()
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    barrier(world)
    torch.cuda.synchronize()
    ms_per_step = max_over_ranks(e0.elapsed_time(e1), world, dev) / args.steps
    total_slices = cfg.nz * (world if mode == "replicas" else 1)
    value = total_slices / (ms_per_step * 1e-3)

    # tuple counts: nominal C(L-1,k) per slice (per q); evaluated = canonical C(m-1,k)
    hist_np = outs[0][0]["histogram"].cpu().numpy() if nzl else np.zeros((0, bins), np.int32)
    m = (hist_np > 0).sum(axis=1)
    if args.enumeration == "dp":  # class terms of the interval DP (m(m+1)/2 per slice), not tuples
        evaluated = int(sum(int(mm) * (int(mm) + 1) // 2 for mm in m))
    elif args.enumeration == "canonical":
        evaluated = int(sum(comb(int(mm) - 1, k) for mm in m if mm >= k + 1))
    else:
        evaluated = nzl * comb(bins - 1, k)
    nominal = nzl * comb(bins - 1, k)
    evaluated *= len(qs)
    nominal *= len(qs)

    kernels, roofline = None, None
    pk_, how = peaks()
    hbm = float(pk_.get("hbm_gbs", HBM_FALLBACK_GBS))
    itemsize = host.itemsize
    step_bytes = n_vox * itemsize + n_vox * len(qs)  # volume once + labels per q (single pass)
    two_pass = n_vox * itemsize * (1 + len(qs)) + n_vox * len(qs)
    kind = tsa.tsa_pipeline_kind(p) if nzl else -1
    if rank == 0 and nzl > 0:
        stt = stage_times(cfg, args, vols, nbuf, dev)
        hist_b, lab_b = n_vox * itemsize, n_vox * (itemsize + 1)
        kernels = {
            "histogram": {"ms": stt["histogram"], "calls_per_step": 1, "bytes": hist_b,
                          "gbs": hist_b / (stt["histogram"] * 1e-3) / 1e9,
                          "frac_hbm": hist_b / (stt["histogram"] * 1e-3) / 1e9 / hbm},
            "search": {"ms": stt["search"], "calls_per_step": len(qs),
                       "note": "k_small_luts + k_scan + [k_k2_seed + k_search_k2 + k_merge_items | k_tri_tables + k_search_tri + k_fold_slots]"},
            "finalize": {"ms": stt["finalize"], "calls_per_step": len(qs)},
            "label": {"ms": stt["label"], "calls_per_step": len(qs), "bytes": lab_b * len(qs),
                      "note": ("the staged per-q label kernel; the sweep step labels all q in one pass "
                               "(k_label_sweep: the volume read once)") if sweep else None,
                      "gbs": lab_b * len(qs) / (stt["label"] * 1e-3) / 1e9,
                      "frac_hbm": lab_b * len(qs) / (stt["label"] * 1e-3) / 1e9 / hbm},
            "per_q": stt["per_q"] if sweep else None,
            "timing": "isolated stage calls captured in CUDA graphs (10 launches x 5 replays), "
                      "the staged kernels; ms = per step (summed over q)",
        }
        fpt = fp64_per_tuple(k, qs[0], args.enumeration)
        peak64, how64 = fp64_peak()
        if fpt is not None:
            ach = evaluated * fpt / (stt["search"] * 1e-3)
            kernels["search"].update({"tuples_evaluated": evaluated, "tuples_nominal": nominal,
                                      "gtuples_per_s_evaluated": evaluated / (stt["search"] * 1e-3) / 1e9,
                                      "gtuples_per_s_nominal": nominal / (stt["search"] * 1e-3) / 1e9,
                                      "fp64_instr_per_tuple": fpt, "fp64_lane_instr_per_s": ach,
                                      "frac_fp64": ach / peak64})
            if args.enumeration == "canonical" and (k >= 3 or (k == 2 and all(q < 1 for q in qs))):
                kernels["search"]["pruning"] = (
                    "exact bounds (DESIGN.md §7b): every canonical tuple is evaluated or excluded by a rigorous "
                    "upper bound below a score already reached, so the result is the exhaustive search's bit for "
                    "bit; tuples_evaluated counts the canonical tuples COVERED and the fp64 rate / frac_fp64 are "
                    "the exhaustive-equivalent rate (covered tuples x the per-tuple instructions of the "
                    "unpruned loop / stage time)")
        tr = {}
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tr = json.load(f).get(args.workload, {})
        dom = max(("histogram", "search", "label"), key=lambda n: kernels[n]["ms"])
        if kind in (2, 3, 4):
            # overlapped pipelines: the product step is one chain of co-resident
            # kernels, timed as a whole against the single-pass HBM floor
            names = {2: "compact step (k_lut_part + k_hist_part + k_mid + k_label_part, PDL-chained)",
                     3: "stream step (k_stream: io + search CTAs, per-slice flags)",
                     4: "overlap step (staged kernels on 8 slabs over two streams: histogram / labels "
                        "of one slab next to the search of another)"}
            ach = step_bytes / (ms_per_step * 1e-3) / 1e9
            roofline = {"bound": "hbm", "kernel": names[kind], "achieved": ach, "peak": hbm, "unit": "GB/s",
                        "frac": ach / hbm, "traffic": tr.get({2: "compact", 3: "stream", 4: "overlap"}[kind]),
                        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({how})",
                        "algorithmic_bytes_per_launch": step_bytes,
                        "note": "timed = the whole step (CUDA events over the timed region / steps); bytes = "
                                "volume once + labels once"}
            if fpt is not None:
                roofline["fp64_search_stage"] = {
                    "frac": kernels["search"]["frac_fp64"], "peak": peak64 / 1e12, "unit": "T FP64 lane-instr/s",
                    "note": "the search of the same step run alone through the staged stage calls"}
        elif dom == "search" and fpt is not None:
            roofline = {"bound": "fp64", "kernel": "search stage (" + kernels["search"]["note"] + ")",
                        "achieved": kernels["search"]["fp64_lane_instr_per_s"] / 1e12, "peak": peak64 / 1e12,
                        "unit": "T FP64 lane-instr/s", "frac": kernels["search"]["frac_fp64"],
                        "traffic": tr.get("search"), "peak_source": how64,
                        "algorithmic_fp64_instr_per_launch": evaluated * fpt / len(qs),
                        "fp64_instr_per_tuple": fpt, "tuples_evaluated_per_launch": evaluated // len(qs)}
        else:
            kd = kernels[dom] if dom != "search" else kernels["histogram"]
            roofline = {"bound": "hbm", "kernel": f"k_{dom}", "achieved": kd["gbs"], "peak": hbm,
                        "unit": "GB/s", "frac": kd["gbs"] / hbm, "traffic": tr.get(dom),
                        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({how})",
                        "algorithmic_bytes_per_launch": kd["bytes"] // kd["calls_per_step"]}
        roofline["step_hbm"] = {
            "single_pass_bytes": step_bytes, "two_pass_bytes": two_pass,
            "achieved_gbs_single_pass": step_bytes / (ms_per_step * 1e-3) / 1e9,
            "frac_single_pass": step_bytes / (ms_per_step * 1e-3) / 1e9 / hbm,
            "frac_two_pass": two_pass / (ms_per_step * 1e-3) / 1e9 / hbm, "peak_gbs": hbm,
            "note": "the whole step (all kernels) against the HBM floor: single pass = volume once + "
                    "labels; two pass = the label pass re-reads the volume"}
        roofline["stage_share_of_step"] = {n: kernels[n]["ms"] / ms_per_step for n in
                                           ("histogram", "search", "finalize", "label")}

    # -------- e2e: host buffers through the public API (copies inside the timed region)
    e2e = None
    if args.e2e_steps > 0 and nzl > 0:
        host_t = torch.from_numpy(host).pin_memory()
        h2d = int(host.nbytes)
        if sweep:
            hout = [{"thresholds": torch.empty((nzl, k), dtype=torch.int32).pin_memory(),
                     "objective": torch.empty(nzl, dtype=torch.float64).pin_memory(),
                     "status": torch.empty(nzl, dtype=torch.int32).pin_memory(),
                     "labels": torch.empty(host.shape, dtype=torch.uint8).pin_memory()} for _ in qs]
            dvol = torch.empty_like(vols[0])

            def e2e_step():
                dvol.copy_(host_t, non_blocking=True)
                tsa.tsa_segment_sweep(dvol, bins, k, qs, enumeration=args.enumeration, outs=outs[0],
                                      workspace=wss, stream=stream)
                for j in range(len(qs)):
                    for key in hout[j]:
                        hout[j][key].copy_(outs[0][j][key], non_blocking=True)
                torch.cuda.synchronize()

            api = "pinned H2D + tsa_segment_sweep (11 q) + D2H of every q's thresholds/objective/status/labels"
            d2h = sum(t.numel() * t.element_size() for h in hout for t in h.values())
        else:
            hout = {"thresholds": torch.empty((nzl, k), dtype=torch.int32).pin_memory(),
                    "objective": torch.empty(nzl, dtype=torch.float64).pin_memory(),
                    "status": torch.empty(nzl, dtype=torch.int32).pin_memory(),
                    "labels": torch.empty(host.shape, dtype=torch.uint8).pin_memory()}
            slab = min(nzl, args.e2e_slab or (50 if bins <= 256 else 25))  # slices per host<->device slab
            hp = tsa.make_problem(host_t, bins, k, qs[0], enumeration=args.enumeration)
            scratch = torch.empty(int(tsa.load().tsa_segment_host_scratch_size(ctypes.byref(hp), slab)),
                                  dtype=torch.uint8, device=dev)
            s2 = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))

            def e2e_step():
                tsa.tsa_segment_host(host_t, bins, k, qs[0], enumeration=args.enumeration, slab=slab,
                                     scratch=scratch, streams=s2, out=hout)

            api = "tsa_segment_host (pinned host buffers, 2-stream slab pipeline)"
            d2h = sum(t.numel() * t.element_size() for t in hout.values())
        for _ in range(2):
            e2e_step()
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        dt = max_over_ranks(time.perf_counter() - t0, world, dev)
        barrier(world)
        e2e = {"value": total_slices * args.e2e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(d2h), "api": api, "steps": args.e2e_steps,
               "note": "per rank" if world > 1 else None}
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, host, qs)

    # our kernels per step: compact k_lut_part + k_hist_part + k_mid + k_label_part;
    # staged k_histogram + per q (k_small_luts + k_scan [+ k_rtable | k_tri_tables]
    # [+ k_k2_seed] + search [+ k_merge_items | k_fold_slots] + [k_decide +] label + k_finalize[_phi])
    rtable = k >= 3 and bins <= 512 and args.enumeration == "full"  # canonical k >= 3: k_search_tri
    tri = k >= 3 and bins <= 512 and args.enumeration == "canonical"  # + k_fold_slots
    # + k_k2_seed: the bounded k = 2 search (q < 1, TSA_K2_PRUNE not 0), fused
    # into k_scan_seed (replacing k_scan) unless TSA_K2_FUSE=0
    seed = k == 2 and args.enumeration == "canonical" and qs[0] < 1 and os.environ.get("TSA_K2_PRUNE", "1")[:1] != "0"
    seed_kernel = seed and os.environ.get("TSA_K2_FUSE", "1")[:1] == "0"
    # staged step with labels: k_decide + labels + k_finalize_phi (split finalize)
    split = not sweep and os.environ.get("TSA_SPLIT_FINALIZE", "1")[:1] != "0"
    per_q = 5 + (1 if rtable else 0) + (1 if k == 2 and args.enumeration != "dp" else 0) + (2 if tri else 0) + \
        (1 if seed_kernel else 0) + (1 if split else 0)
    slabs = min(cfg.nz, 8)
    if sweep:  # one histogram, per q the search chain, one k_label_sweep per 16 q
        launches_per_step = 1 + (per_q - 1) * len(qs) + -(-len(qs) // 16)
    else:
        launches_per_step = {1: 1, 2: 4, 3: 2, 4: slabs * (1 + per_q)}.get(kind, 1 + per_q)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if mode == "replicas" else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_of(cfg, args, world),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "kernels": kernels, "pipeline": {1: "fused", 2: "compact", 3: "stream", 4: "overlap"}.get(kind, "staged"),
            "gtuples_per_s_nominal": cfg.nz * comb(bins - 1, k) * len(qs) * (world if mode == "replicas" else 1)
                                     / (ms_per_step * 1e-3) / 1e9,
            "gtuples_per_s_evaluated": evaluated * total_slices / max(nzl, 1) / (ms_per_step * 1e-3) / 1e9,
            "slice_q_pairs_per_s": value * len(qs) if sweep else None,
            "provenance": provenance(cfg, host, dev) if nzl else None,
        }
        print(json.dumps(line), flush=True)


def run_tuple_sharded(args, cfg, rank, world, dev):
    """One volume, tuple space of every slice split over the ranks (SURVEY.md
    §8(e), config c4) through tsa_segment_sharded: NCCL all-gathers of the
    histograms and of the (score, key) partials inside libtsa, labels of the
    own slab.  value = nz / max-over-ranks device time (strong scaling)."""
    from math import comb

    import numpy as np
    import torch

    import phantom
    import paper_2012_10684_b200 as tsa
    from paper_2012_10684_b200.dist import make_comm

    import torch.distributed as dist

    if world == 1 and not dist.is_initialized():
        import socket

        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        dist.init_process_group("nccl", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}",
                                device_id=dev)
    q = cfg.qs[0]
    z0, z1 = tsa.tsa_slab_range(cfg.nz, world, rank)
    host = phantom.make_volume(cfg, nz=z1 - z0, z_first=z0) if z1 > z0 else \
        np.zeros((0, cfg.ny, cfg.nx), cfg.np_dtype)
    slab = torch.from_numpy(np.ascontiguousarray(host)).to(dev)
    comm = make_comm(None, dev)
    p = tsa.tsa_problem(slab.data_ptr() if z1 > z0 else None, 1 if cfg.dtype == "u8" else 2, cfg.nx, cfg.ny,
                        z1 - z0, cfg.bins, cfg.k, q, 0, tsa.ENUMERATIONS[args.enumeration], 0, 0, 0, 0)
    import ctypes

    ws = torch.empty(max(1, int(tsa.load().tsa_sharded_workspace_size(ctypes.byref(p), cfg.nz, 1,
                                                                       comm.handle))),
                     dtype=torch.uint8, device=dev)

    def step():
        return tsa.tsa_segment_sharded(slab, cfg.nz, cfg.bins, cfg.k, q, comm, mode="tuples",
                                       enumeration=args.enumeration, workspace=ws, nx=cfg.nx, ny=cfg.ny)

    sampler = ClockSampler(dev.index)
    sampler.start()
    for _ in range(max(args.warmup, 3)):
        out = step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.perf_counter()
    e0.record()
    for _ in range(args.steps):
        out = step()
    e1.record()
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    dist.barrier()
    ms_step = max_over_ranks(e0.elapsed_time(e1), world, dev) / args.steps
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)
    hist = out["histogram"].cpu().numpy()
    m = (hist > 0).sum(axis=1)
    if args.enumeration == "dp":  # class terms of the interval DP, not tuples
        evaluated = int(sum(int(x) * (int(x) + 1) // 2 for x in m))
    elif args.enumeration == "canonical":
        evaluated = int(sum(comb(int(x) - 1, cfg.k) for x in m if x >= cfg.k + 1))
    else:
        evaluated = cfg.nz * comb(cfg.bins - 1, cfg.k)
    if rank == 0:
        line = {
            "metric": METRIC, "value": cfg.nz / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(cfg, args, world), "clocks": clocks,
            "gtuples_per_s_nominal": cfg.nz * comb(cfg.bins - 1, cfg.k) / (ms_step * 1e-3) / 1e9,
            "gtuples_per_s_evaluated": evaluated / (ms_step * 1e-3) / 1e9,
            "gpu_launches": None, "units": out["units"], "comm": {1: "nccl", 2: "custom"}[comm.kind],
            "roofline": None, "cpu_baseline": None, "e2e": None,
            "note": "kernels per step: histogram, small LUT, scan, [R table], search, merge, fill/none, "
                    "finalize, label + 4 NCCL all-gathers",
        }
        print(json.dumps(line), flush=True)
    comm.close()


def dry_run(args):
    """Launcher check without a GPU (tests/test_bench_contract.py): every rank
    joins a gloo group and rank 0 prints the JSON shape with n_gpus = world."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.zeros(world, dtype=torch.int64)
        t[rank] = rank + 1
        dist.all_reduce(t)
        ranks = [int(x) - 1 for x in t]
        dist.destroy_process_group()
    else:
        ranks = [0]
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "ranks": ranks,
                          "dry_run": True, "workload": args.workload}), flush=True)


def spawn_ranks(args):
    """bench.py --gpus N outside torchrun: re-launch under torch.distributed.run
    with N local ranks (127.0.0.1 rendezvous) and return its exit code."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.dry_run:
        dry_run(args)
        return
    import phantom

    cfg = phantom.CONFIGS[args.workload]
    if args.impl == "reference":
        if world > 1 and rank != 0:
            return
        run_reference(args, cfg, rank, world)
        return

    import torch

    import paper_2012_10684_b200 as tsa

    tsa.load()  # fails loudly if the CUDA library is missing: no fallback
    assert torch.cuda.is_available(), "bench needs a GPU"
    # TSA_BENCH_ONE_GPU=1 (tests only): every rank on cuda:0 over gloo, to run
    # the multi-rank flow on a one-GPU box; NCCL (one GPU per rank) otherwise
    one_gpu = os.environ.get("TSA_BENCH_ONE_GPU") == "1"
    local = 0 if one_gpu else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    try:
        if cfg.name in ("c1", "c2", "c3", "c4", "c5") and shard_mode(args, cfg, world) == "tuples":
            run_tuple_sharded(args, cfg, rank, world, dev)
        elif cfg.name == "f1":
            run_2d(args, cfg, rank, world, dev)
        elif cfg.name == "f2":
            run_hu(args, cfg, rank, world, dev)
        elif cfg.name == "f3":
            run_morph(args, cfg, rank, world, dev)
        else:
            run_1d(args, cfg, rank, world, dev)
    finally:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
