"""Multi-GPU execution of the hot path ("job
distribution ... reduction of results from different devices").

One process per GPU, torch.distributed process group (NCCL over NVLink on the
B200 box; gloo for the CPU tests of the host logic).  Two strategies:

* slab sharding (``segment_slabs``): rank r segments slices
  [slab_range(nz, P, r)) with no data-path collective -- slices are
  independent problems.
* tuple sharding (``segment_tuple_sharded`` -> the library's
  ``tsa_segment_sharded``, NCCL inside libtsa): every rank needs the same
  per-slice argmax over a tuple space too large for one GPU (k = 4).  Each rank
  histograms its slab, the histograms are all-gathered (nz*L*4 bytes), each
  rank runs the exhaustive search over its share of the work units of *every*
  slice, the per-slice (score, key) partials are all-gathered (16 B per slice
  per rank) and merged under the total order (score desc, key asc) by
  ``tsa_finalize``.  The unit partition is rank-independent, so the result is
  bit-identical to the 1-GPU result for any world size.

The collectives move only small host-independent tensors; every step of the
path itself runs in the libtsa kernels.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

from . import (TsaComm, tsa_comm_unique_id, tsa_default_units, tsa_finalize, tsa_histogram,
               tsa_hu_finish, tsa_hu_histogram, tsa_label, tsa_merge, tsa_search, tsa_segment,
               tsa_segment_sharded, ENUMERATIONS)


def slab_range(nz: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slab [z0, z1) of rank `rank`: ceil(nz/P) slices per rank,
    the last ranks possibly fewer (or none)."""
    per = -(-nz // world)
    z0 = min(nz, rank * per)
    return z0, min(nz, z0 + per)


def unit_range(units: int, world: int, rank: int) -> tuple[int, int]:
    """Work units [u0, u1) of rank `rank` out of `units` per slice (balanced,
    disjoint, covering)."""
    return units * rank // world, units * (rank + 1) // world


def _all_gather(out: torch.Tensor, inp: torch.Tensor, group=None):
    """all_gather_into_tensor; gloo cannot gather CUDA tensors, so route them
    through host memory there (tests only: NCCL is the production backend)."""
    if inp.is_cuda and dist.get_backend(group) == "gloo":
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)


def gather_rows(local: torch.Tensor, rows_per_rank: int, group=None) -> torch.Tensor:
    """All-gather equally sized row blocks (rank-major).  `local` is padded to
    `rows_per_rank` rows with zeros; returns [world * rows_per_rank, ...]."""
    world = dist.get_world_size(group)
    if local.shape[0] < rows_per_rank:
        pad = torch.zeros((rows_per_rank - local.shape[0],) + tuple(local.shape[1:]),
                          dtype=local.dtype, device=local.device)
        local = torch.cat([local, pad])
    out = torch.empty((world * rows_per_rank,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    _all_gather(out, local.contiguous(), group)
    return out


def gather_partials(score: torch.Tensor, key: torch.Tensor, group=None):
    """All-gather per-slice partial argmax results: [nz] -> [world, nz]."""
    world = dist.get_world_size(group)
    n = score.shape[0]
    s = torch.empty(world * n, dtype=score.dtype, device=score.device)
    k = torch.empty(world * n, dtype=key.dtype, device=key.device)
    _all_gather(s, score.contiguous(), group)
    _all_gather(k, key.contiguous(), group)
    return s.view(world, n), k.view(world, n)


def agreed_units(nz_total, bins, k, enum, world, units=0, group=None, device=None) -> int:
    """Work units per slice, identical on every rank.  The library heuristic
    depends on the local SM count, so every rank proposes its value and the
    group takes the maximum (one tiny all-reduce): unit_range() then
    partitions the same unit space on every rank even on mixed devices.  The
    interval DP has exactly one unit per slice (tsa_search rejects more)."""
    if enum == ENUMERATIONS["dp"]:
        return 1
    if units > 0:
        return units
    U = max(world, tsa_default_units(nz_total, bins, k, enum))
    if world > 1:
        t = torch.tensor([U], dtype=torch.int64,
                         device=device if dist.get_backend(group) != "gloo" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        U = int(t.item())
    return U


def segment_slabs(vol_slab, bins, k, q, **kw):
    """Slab sharding: this rank's slices only, no collective."""
    return tsa_segment(vol_slab, bins, k, q, **kw)


_cudart = None


def _cudart_lib():
    """libcudart for the host staging of the gloo transport (tests only)."""
    global _cudart
    if _cudart is None:
        import ctypes

        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                _cudart = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if _cudart is None:
            import glob

            cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime",
                                           "lib", "libcudart.so*"))
            _cudart = ctypes.CDLL(cands[0])
    return _cudart


def _gloo_allgather(group):
    """All-gather for tsa_comm_init_custom over a gloo group: synchronise the
    library's stream, stage the rank's bytes through host memory, gather,
    copy the rank-major result back.  Two ranks on one GPU (NCCL refuses)
    and CPU-side tests use it; the product transport is NCCL."""
    import ctypes

    import numpy as np

    rt = _cudart_lib()
    rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    rt.cudaStreamSynchronize.argtypes = [ctypes.c_void_p]

    def fn(send, recv, nbytes, stream):
        world = dist.get_world_size(group)
        if rt.cudaStreamSynchronize(stream) != 0:
            raise RuntimeError("cudaStreamSynchronize")
        mine = np.empty(nbytes, np.uint8)
        if nbytes and rt.cudaMemcpy(mine.ctypes.data, send, nbytes, 2) != 0:  # D2H
            raise RuntimeError("cudaMemcpy D2H")
        out = torch.empty(world * nbytes, dtype=torch.uint8)
        dist.all_gather_into_tensor(out, torch.from_numpy(mine), group=group)
        o = out.numpy()
        if nbytes and rt.cudaMemcpy(recv, o.ctypes.data, world * nbytes, 1) != 0:  # H2D
            raise RuntimeError("cudaMemcpy H2D")

    return fn


def make_comm(group=None, device=None):
    """A libtsa communicator over the ranks of `group`: NCCL (tsa_comm_init,
    the unique id broadcast from rank 0 through the process group) when the
    group's backend is NCCL, else the host-staged gloo all-gather."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if dist.get_backend(group) == "nccl":
        uid = [tsa_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0, group=group, device=device)
        return TsaComm.nccl(world, rank, uid[0])
    return TsaComm.custom(world, rank, _gloo_allgather(group))


def segment_tuple_sharded(vol_slab, nz_total, bins, k, q, objective="pseudo_additive",
                          enumeration="canonical", units=0, group=None, labels=True,
                          workspace=None, comm=None):
    """Tuple sharding across the group through the library
    (tsa_segment_sharded, TSA_SHARD_TUPLES): `vol_slab` is this rank's slab
    (slab_range(nz_total, P, rank)) on this rank's GPU.  Returns the full
    per-slice results (thresholds/objective/status/histogram for all nz_total
    slices, identical on every rank) and this rank's labels."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    own = comm is None
    if own:
        comm = make_comm(group, vol_slab.device)
    try:
        out = tsa_segment_sharded(vol_slab, nz_total, bins, k, q, comm, mode="tuples",
                                  objective=objective, enumeration=enumeration, units=units,
                                  labels=labels, workspace=workspace)
    finally:
        if own:
            comm.close()
    U = out["units"]
    out["unit_range"] = unit_range(U, world, rank)
    out["slab"] = slab_range(nz_total, world, rank)
    return out


def segment_tuple_sharded_py(vol_slab, nz_total, bins, k, q, objective="pseudo_additive",
                             enumeration="canonical", units=0, group=None, labels=True,
                             workspace=None):
    """The same exchange driven from Python with torch.distributed collectives
    around the stage calls (kept as a cross-check of the in-library path)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-nz_total // world)
    dev = vol_slab.device
    if vol_slab.shape[0] > 0:
        hist_l, st_l = tsa_histogram(vol_slab, bins)
    else:
        hist_l = torch.zeros((0, bins), dtype=torch.int32, device=dev)
        st_l = torch.zeros(0, dtype=torch.int32, device=dev)
    hist = gather_rows(hist_l, per, group)[:nz_total].contiguous()
    status = gather_rows(st_l, per, group)[:nz_total].contiguous()
    enum = ENUMERATIONS.get(enumeration, enumeration)
    U = agreed_units(nz_total, bins, k, enum, world, units, group, dev)
    u0, u1 = unit_range(U, world, rank)
    if u1 > u0:
        ps, pk = tsa_search(hist, status, vol_slab.shape[1] * vol_slab.shape[2], k, q, objective,
                            enumeration, units=U, unit_begin=u0, unit_end=u1, workspace=workspace)
        s_loc, k_loc = tsa_merge(ps, pk)
    else:  # more ranks than units: contribute "no tuple"
        s_loc = torch.full((nz_total,), float("-inf"), dtype=torch.float64, device=dev)
        k_loc = torch.full((nz_total,), -1, dtype=torch.int64, device=dev)
    ps_all, pk_all = gather_partials(s_loc, k_loc, group)
    thr, phi, st = tsa_finalize(hist, status, k, q, ps_all, pk_all, objective=objective)
    z0, z1 = slab_range(nz_total, world, rank)
    lab = None
    if labels and z1 > z0:
        lab = tsa_label(vol_slab, thr[z0:z1].contiguous(), st[z0:z1].contiguous(), bins=bins)
    return {"thresholds": thr, "objective": phi, "status": st, "histogram": hist, "labels": lab,
            "units": U, "unit_range": (u0, u1), "slab": (z0, z1)}


INT32_MAX, INT32_MIN = 2**31 - 1, -2**31


def reduce_window(win: torch.Tensor, group=None) -> torch.Tensor:
    """Volume-wide HU window from every rank's slab window (lo, hi): one
    all-reduce MIN of (lo, -hi) (an all-background slab contributes the
    neutral (INT32_MAX, INT32_MIN)).  The only exchange of the HU path."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return win
    t = torch.stack([win[0].to(torch.int64), -win[1].to(torch.int64)])
    if dist.get_backend(group) == "gloo":  # (CPU tests; NCCL reduces on the device)
        t = t.cpu()
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return torch.stack([t[0], -t[1]]).to(torch.int32).to(win.device)


def hu_segment_slabs(vol_slab, k, q, background=-2000, group=None, **kw):
    """HU path with slices sharded over ranks (SURVEY.md §8(e) + §8(f) row 2):
    phase 1 on the own slab, the window all-reduce, phase 2.  Bit-identical
    to the single-GPU tsa_hu_segment of the whole volume."""
    dev = vol_slab.device
    if vol_slab.shape[0] > 0:
        win, ws = tsa_hu_histogram(vol_slab, k, q, background, **kw)
    else:  # an empty slab still takes part in the exchange
        win, ws = torch.tensor([INT32_MAX, INT32_MIN], dtype=torch.int32, device=dev), None
    wall = reduce_window(win, group)
    if vol_slab.shape[0] == 0:
        return {"window": wall}
    out = tsa_hu_finish(vol_slab, k, q, wall.to(dev).contiguous(), ws, background, **kw)
    out["window"] = wall
    return out
