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
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--impl", default="tsa", choices=["tsa", "reference"])
    ap.add_argument("--enumeration", default="canonical", choices=["canonical", "full", "dp"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--buffers", type=int, default=0, help="resident volume copies rotated (0 = auto, > 2x L2)")
    ap.add_argument("--shard", default="slices", choices=["slices", "tuples"],
                    help="slices: every rank segments its own volume (weak scaling); tuples: the "
                         "ranks split the tuple space of one volume, NCCL all-gathers (strong)")
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

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def cpu_baseline(cfg, vol, q, target_s=10.0):
    """The oracle as it stands, on the host cores, over a bounded sample of the
    workload: whole-volume passes (or a slice prefix) repeated until about
    target_s seconds of wall time (capped at 20 passes)."""
    import oracle

    threads = oracle.max_threads()
    n0 = min(cfg.nz, max(threads, 4))
    t = time.perf_counter()
    oracle.segment(vol[:n0], cfg.bins, cfg.k, q, threads=threads)
    dt = time.perf_counter() - t
    n = int(min(cfg.nz, max(n0, n0 * target_s / max(dt, 1e-6))))
    reps, slices, t = 0, 0, time.perf_counter()
    while True:
        oracle.segment(vol[:n], cfg.bins, cfg.k, q, threads=threads)
        reps += 1
        slices += n
        el = time.perf_counter() - t
        if el >= target_s or reps >= 20:
            break
    return {"value": slices / el, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{reps} pass(es) over the first {n} of {cfg.nz} slices of workload {cfg.name} "
                      f"(whole path: histogram, exhaustive Level-1 search, labels), {threads} OpenMP "
                      f"threads, {el:.2f} s"}


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
    q = cfg.qs[0]
    vol = phantom.make_volume(cfg)
    threads = oracle.max_threads()
    if cfg.name == "f2":  # HU input: the pre-processing oracle, then the 1-D oracle
        def seg(v, bins, k, q_, threads=None):
            g, _, _ = oracle.preprocess(v)
            return oracle.segment(g, 256, k, q_, threads=threads)
        what = "pre-processing + whole 1-D path"
    elif cfg.name == "f3":  # disk(10) top-hat, brute force
        def seg(v, bins, k, q_, threads=None):
            return oracle.tophat(v, cfg.k)
        what = f"brute-force disk({cfg.k}) opening + top-hat, single-threaded"
    else:
        seg = oracle.segment
        what = "whole path, Level-1 oracle"
    t = time.perf_counter()
    seg(vol[:threads], cfg.bins, cfg.k, q, threads=threads)
    per_slice = (time.perf_counter() - t) / threads
    budget = 120.0
    spp = int(max(1, min(cfg.nz, budget / max(args.steps + args.warmup, 1) / max(per_slice, 1e-6))))
    z = 0
    for _ in range(args.warmup):
        seg(vol[z:z + spp], cfg.bins, cfg.k, q, threads=threads)
    t = time.perf_counter()
    for s in range(args.steps):
        z0 = (s * spp) % max(1, cfg.nz - spp + 1)
        seg(vol[z0:z0 + spp], cfg.bins, cfg.k, q, threads=threads)
    dt = time.perf_counter() - t
    value = spp * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_for(cfg, args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{spp} slices of {cfg.name} per step ({what})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
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


def config_of(cfg, args, world):
    return {"workload": f"{cfg.name}: {cfg.note}", "nx": cfg.nx, "ny": cfg.ny,
            "slices_per_gpu": cfg.nz, "bins": cfg.bins, "k": cfg.k, "q": cfg.qs[0],
            "input": cfg.dtype, "objective": "pseudo_additive", "enumeration": args.enumeration,
            "parallelism": f"slices sharded, {world} GPU(s), no collective",
            "l2": "inputs larger than L2: rotating resident volume/label copies (> 2x 126 MB)"}


def run_tuple_sharded(args, cfg, rank, world, dev):
    """One volume, tuple space split over the ranks:
    histogram all-gather, per-rank search over its work units of every slice,
    (score, key) all-gather, merge/finalize, labels of the own slab."""
    import numpy as np
    import torch

    import phantom
    import paper_2012_10684_b200 as tsa
    from paper_2012_10684_b200.dist import segment_tuple_sharded, slab_range

    if world > 1:
        import torch.distributed as dist
    else:
        import torch.distributed as dist

        import socket

        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        dist.init_process_group("gloo", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
    q = cfg.qs[0]
    z0, z1 = slab_range(cfg.nz, world, rank)
    host = phantom.make_volume(cfg, nz=z1 - z0, z_first=z0) if z1 > z0 else \
        np.zeros((0, cfg.ny, cfg.nx), cfg.np_dtype)
    slab = torch.from_numpy(np.ascontiguousarray(host)).to(dev)
    ws = None
    for _ in range(max(args.warmup, 3)):
        segment_tuple_sharded(slab, cfg.nz, cfg.bins, cfg.k, q, enumeration=args.enumeration)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        out = segment_tuple_sharded(slab, cfg.nz, cfg.bins, cfg.k, q, enumeration=args.enumeration)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = max_over_ranks(e0.elapsed_time(e1), world, dev) if world > 1 else e0.elapsed_time(e1)
    ms_step = ms / args.steps
    from math import comb

    hist = out["histogram"].cpu().numpy()
    m = (hist > 0).sum(axis=1)
    evaluated = int(sum(comb(int(x) - 1, cfg.k) for x in m)) if args.enumeration == "canonical" \
        else cfg.nz * comb(cfg.bins - 1, cfg.k)
    if rank == 0:
        line = {
            "metric": METRIC, "value": cfg.nz / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_of(cfg, args, world),
                           parallelism=f"tuple space of every slice split over {world} GPU(s); "
                                       "NCCL all-gather of histograms and (score, key) partials"),
            "gtuples_per_s_nominal": cfg.nz * comb(cfg.bins - 1, cfg.k) / (ms_step * 1e-3) / 1e9,
            "gtuples_per_s_evaluated": evaluated / (ms_step * 1e-3) / 1e9,
            "gpu_launches": None, "units": out["units"],
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    import phantom

    cfg = phantom.CONFIGS[args.workload]
    rank, world, local = dist_env()
    if args.impl == "reference":
        if world > 1 and rank != 0:
            return
        run_reference(args, cfg, rank, world)
        return

    import numpy as np
    import torch

    import paper_2012_10684_b200 as tsa

    assert torch.cuda.is_available(), "bench needs a GPU"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    if args.shard == "tuples":
        run_tuple_sharded(args, cfg, rank, world, dev)
        return
    if cfg.name == "f1":
        run_2d(args, cfg, rank, world, dev)
        return
    if cfg.name == "f2":
        run_hu(args, cfg, rank, world, dev)
        return
    if cfg.name == "f3":
        run_morph(args, cfg, rank, world, dev)
        return
    q = cfg.qs[0]
    k, bins = cfg.k, cfg.bins
    host = phantom.make_volume(cfg)
    vol_bytes = host.nbytes
    n_vox = host.size
    # resident copies so that consecutive steps never hit L2 (126 MB)
    nbuf = args.buffers or max(2, int(np.ceil(2 * 126e6 / (vol_bytes + n_vox))) + 1)
    vols = [torch.from_numpy(host).to(dev) for _ in range(nbuf)]
    p = tsa.make_problem(vols[0], bins, k, q, enumeration=args.enumeration, pipeline=args.pipeline)
    ws = tsa.workspace_for(p, dev)
    outs = []
    for i in range(nbuf):
        outs.append({
            "thresholds": torch.empty((cfg.nz, k), dtype=torch.int32, device=dev),
            "objective": torch.empty(cfg.nz, dtype=torch.float64, device=dev),
            "histogram": torch.empty((cfg.nz, bins), dtype=torch.int32, device=dev),
            "status": torch.empty(cfg.nz, dtype=torch.int32, device=dev),
            "labels": torch.empty(host.shape, dtype=torch.uint8, device=dev),
        })
    stream = torch.cuda.current_stream()

    def step(i):
        tsa.tsa_segment(vols[i % nbuf], bins, k, q, enumeration=args.enumeration, out=outs[i % nbuf],
                        workspace=ws, stream=stream, pipeline=args.pipeline)

    sampler = ClockSampler(local)
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
    ms = e0.elapsed_time(e1)
    ms_max = max_over_ranks(ms, world, dev)
    ms_per_step = ms_max / args.steps
    value = world * cfg.nz / (ms_per_step * 1e-3)

    # -------- per-kernel timing pass (same kernels through the stage calls)
    nvox_slice = cfg.nx * cfg.ny
    U = tsa.tsa_default_units(cfg.nz, bins, k, args.enumeration)
    hist = torch.empty((cfg.nz, bins), dtype=torch.int32, device=dev)
    st = torch.empty(cfg.nz, dtype=torch.int32, device=dev)
    sws = torch.empty(tsa.tsa_search_workspace_size(cfg.nz, nvox_slice, bins, k, q, 0, args.enumeration),
                      dtype=torch.uint8, device=dev)
    reps = max(20, min(args.steps, 400))
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(reps)]
    for i in range(reps + 3):
        j = i - 3
        v = vols[i % nbuf]
        if j >= 0:
            ev[j][0].record(stream)
        h, s = tsa.tsa_histogram(v, bins)
        if j >= 0:
            ev[j][1].record(stream)
        ps, pk = tsa.tsa_search(h, s, nvox_slice, k, q, enumeration=args.enumeration, units=U,
                                workspace=sws)
        if j >= 0:
            ev[j][2].record(stream)
        thr, phi, st2 = tsa.tsa_finalize(h, s, k, q, ps, pk)
        if j >= 0:
            ev[j][3].record(stream)
        tsa.tsa_label(v, thr, st2, bins=bins)
        if j >= 0:
            ev[j][4].record(stream)
    torch.cuda.synchronize()
    stage_ms = {}
    for si, name in enumerate(["histogram", "search", "finalize", "label"]):
        stage_ms[name] = statistics.mean(ev[j][si].elapsed_time(ev[j][si + 1]) for j in range(reps))
    hist_bytes = n_vox * host.itemsize
    label_bytes = n_vox * (host.itemsize + 1)
    kernels = {
        "histogram": {"ms": stage_ms["histogram"], "bytes": hist_bytes,
                      "gbs": hist_bytes / (stage_ms["histogram"] * 1e-3) / 1e9},
        "search": {"ms": stage_ms["search"] + stage_ms["finalize"]},
        "label": {"ms": stage_ms["label"], "bytes": label_bytes,
                  "gbs": label_bytes / (stage_ms["label"] * 1e-3) / 1e9},
    }
    # tuple counts: nominal C(L-1,k) per slice; evaluated = canonical C(m-1,k)
    from math import comb

    hist_np = outs[0]["histogram"].cpu().numpy()
    m = (hist_np > 0).sum(axis=1)
    if args.enumeration == "dp":  # class terms of the interval DP (m(m+1)/2 per slice), not tuples
        evaluated = int(sum(int(mm) * (int(mm) + 1) // 2 for mm in m))
    else:
        evaluated = int(sum(comb(int(mm) - 1, k) for mm in m)) if args.enumeration == "canonical" else \
            cfg.nz * comb(bins - 1, k)
    nominal = cfg.nz * comb(bins - 1, k)
    kernels["search"]["tuples_nominal"] = nominal
    kernels["search"]["tuples_evaluated"] = evaluated
    kernels["search"]["gtuples_per_s_nominal"] = nominal / (kernels["search"]["ms"] * 1e-3) / 1e9
    kernels["search"]["gtuples_per_s_evaluated"] = evaluated / (kernels["search"]["ms"] * 1e-3) / 1e9

    pk_, how = peaks()
    hbm = float(pk_.get("hbm_gbs", HBM_FALLBACK_GBS))
    kind = tsa.tsa_pipeline_kind(p)
    step_bytes = n_vox * (host.itemsize + 1)  # read the volume once + write the labels once
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tr = {}
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f).get(args.workload, {})
    if kind in (1, 2):
        # fused (one persistent kernel) or compact (3 kernels): time each call
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(reps)]
        for i in range(reps + 3):
            if i >= 3:
                evs[i - 3][0].record(stream)
            step(i)
            if i >= 3:
                evs[i - 3][1].record(stream)
        torch.cuda.synchronize()
        fused_ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
        kernels["fused"] = {"ms": fused_ms, "bytes": step_bytes,
                            "gbs": step_bytes / (fused_ms * 1e-3) / 1e9,
                            "note": ("k_fused (+ counter memset)" if kind == 1 else
                                     "k_hist_part + k_mid + k_label_flat") +
                                    "; bytes = volume once + labels once (the re-read is served by L2)"}
        dom = "fused"
        traffic = tr.get("fused") if kind == 1 else tr.get("compact")
    else:
        dom = max(("histogram", "label", "search"), key=lambda nme: kernels[nme]["ms"])
        traffic = tr.get(dom)
    if dom == "search":
        roofline = {"bound": "fp64", "kernel": "k_search", "achieved": None, "peak": None,
                    "unit": "FP64 instr/s", "frac": None, "traffic": traffic,
                    "note": "search-dominated workload: see kernels.search and profiles/"}
    else:
        kname = {"fused": "k_fused" if kind == 1 else "compact step (k_hist_part + k_mid + k_label_flat)"}.get(
            dom, f"k_{dom}")
        roofline = {"bound": "hbm", "kernel": kname, "achieved": kernels[dom]["gbs"], "peak": hbm,
                    "unit": "GB/s", "frac": kernels[dom]["gbs"] / hbm, "traffic": traffic,
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({how})",
                    "algorithmic_bytes_per_launch": kernels[dom]["bytes"]}
    kernels["staged_note"] = "histogram/search/label rows time the one-kernel-per-stage calls"

    # -------- e2e: host buffers through the C ABI (copies inside the timed region)
    e2e = None
    if args.e2e_steps > 0:
        host_t = torch.from_numpy(host).pin_memory()
        hout = {
            "thresholds": torch.empty((cfg.nz, k), dtype=torch.int32).pin_memory(),
            "objective": torch.empty(cfg.nz, dtype=torch.float64).pin_memory(),
            "status": torch.empty(cfg.nz, dtype=torch.int32).pin_memory(),
            "labels": torch.empty(host.shape, dtype=torch.uint8).pin_memory(),
        }
        slab = 50  # slices per host<->device slab (tools/exp_e2e.py)
        hp = tsa.make_problem(host_t, bins, k, q, enumeration=args.enumeration)
        import ctypes

        scratch = torch.empty(int(tsa.load().tsa_segment_host_scratch_size(ctypes.byref(hp), slab)),
                              dtype=torch.uint8, device=dev)
        s2 = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        for _ in range(2):
            tsa.tsa_segment_host(host_t, bins, k, q, enumeration=args.enumeration, slab=slab,
                                 scratch=scratch, streams=s2, out=hout)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            tsa.tsa_segment_host(host_t, bins, k, q, enumeration=args.enumeration, slab=slab,
                                 scratch=scratch, streams=s2, out=hout)
        dt = time.perf_counter() - t0
        dt = max_over_ranks(dt, world, dev)
        barrier(world)
        d2h = sum(t.numel() * t.element_size() for t in hout.values())
        e2e = {"value": world * cfg.nz * args.e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(host.nbytes), "d2h_bytes_per_step": int(d2h),
               "api": "tsa_segment_host (pinned host buffers, 2-stream slab pipeline)",
               "steps": args.e2e_steps}
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, host, q)

    # our kernels per step: fused k_fused; compact k_lut_part + k_hist_part +
    # k_mid + k_label_part; staged k_histogram + k_luts + k_scan [+ k_rtable]
    # + search + k_finalize + label (the DP has no R table)
    rtable = k >= 3 and bins <= 512 and args.enumeration != "dp"
    launches_per_step = {1: 1, 2: 4}.get(kind, 6 + (1 if rtable else 0))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(cfg, args, world),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "kernels": kernels, "pipeline": {1: "fused", 2: "compact"}.get(kind, "staged"),
            "gtuples_per_s_nominal": world * nominal / (ms_per_step * 1e-3) / 1e9,
            "gtuples_per_s_evaluated": world * evaluated / (ms_per_step * 1e-3) / 1e9,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
