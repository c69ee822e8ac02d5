"""Multi-process host logic of the multi-GPU path on CPU (gloo, world_size 2):
slab / unit partitions, the rank-major gathers, and the tuple-sharded argmax
merge (score desc, key asc) reproducing the single-process result.  The GPU
kernels are replaced by a CPU evaluation of the same scores (test-only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2012_10684_b200.dist import gather_partials, gather_rows, slab_range, unit_range

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nz", [1, 7, 300, 301])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_slab_partition_covers(nz, world):
    seen = []
    for r in range(world):
        z0, z1 = slab_range(nz, world, r)
        assert 0 <= z0 <= z1 <= nz
        seen.extend(range(z0, z1))
    assert seen == list(range(nz))


@pytest.mark.parametrize("units", [1, 5, 64, 1184])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_unit_partition_covers(units, world):
    seen = []
    for r in range(world):
        u0, u1 = unit_range(units, world, r)
        seen.extend(range(u0, u1))
    assert seen == list(range(units))


def _score_key(hist, k, q, t):
    """CPU stand-in for the kernel's (score, key): the oracle objective (a
    monotone score) and the packed-threshold key."""
    v = oracle.phi_at(hist, k, q, t)
    if v is None:
        return -np.inf, 0xFFFFFFFFFFFFFFFF
    key = 0
    for x in t:
        key = (key << 12) | int(x)
    return v, key


def _worker(rank, world, port, hists, k, q, units, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import itertools

        nz, L = hists.shape
        # slab-sharded histogram rows, gathered rank-major
        z0, z1 = slab_range(nz, world, rank)
        per = -(-nz // world)
        local = torch.from_numpy(hists[z0:z1].astype(np.int32))
        full = gather_rows(local, per)[:nz].numpy()
        assert (full == hists).all()
        # tuple sharding: this rank's units of every slice
        u0, u1 = unit_range(units, world, rank)
        s_loc = np.full(nz, -np.inf)
        k_loc = np.full(nz, -1, dtype=np.int64)
        NONE = 2**64 - 1
        for z in range(nz):
            tuples = list(itertools.combinations(range(L - 1), k))
            T = len(tuples)
            bv, bk = -np.inf, NONE
            for u in range(u0, u1):
                for t in tuples[T * u // units: T * (u + 1) // units]:
                    v, key = _score_key(hists[z], k, q, t)
                    if v > bv or (v == bv and key < bk):
                        bv, bk = v, key
            s_loc[z] = bv
            k_loc[z] = bk if bk != NONE else -1
        s_all, k_all = gather_partials(torch.from_numpy(s_loc), torch.from_numpy(k_loc))
        # merge under (score desc, key asc): what tsa_finalize does on the GPU
        res = []
        for z in range(nz):
            best = (-np.inf, 2**64 - 1)
            for r in range(world):
                v = s_all[r, z].item()
                kk = int(k_all[r, z].item()) & 0xFFFFFFFFFFFFFFFF
                if v > best[0] or (v == best[0] and kk < best[1]):
                    best = (v, kk)
            res.append(best[1])
        if rank == 0:
            ret.extend(res)
    finally:
        dist.destroy_process_group()


def _tuple_of(key, k):
    return tuple((key >> (12 * (k - 1 - j))) & 0xFFF for j in range(k))


@pytest.mark.parametrize("world", [2])
def test_tuple_sharded_argmax_matches_single_process(world):
    rng = np.random.default_rng(3)
    nz, L, k, q = 3, 10, 2, 0.8
    hists = rng.integers(0, 30, size=(nz, L))
    hists[:, ::4] = 0
    mgr = mp.Manager()
    ret = mgr.list()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, hists, k, q, 5, ret), nprocs=world, join=True)
    for z in range(nz):
        ref = oracle.search(hists[z], k, q)
        assert _tuple_of(ret[z], k) == ref["t"]


def _win_worker(rank, world, port, wins, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    from paper_2012_10684_b200.dist import reduce_window

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ret[rank] = reduce_window(torch.tensor(wins[rank], dtype=torch.int32)).tolist()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_hu_window_allreduce(world):
    """The HU path's only exchange: the volume-wide window of the ranks' slab
    windows (oracle.preprocess on the whole volume is the reference); a slab
    with only background contributes the neutral (INT32_MAX, INT32_MIN)."""
    rng = np.random.default_rng(world)
    vol = rng.integers(-1200, 900, size=(7, 8, 8)).astype(np.int16)
    vol[rng.random(vol.shape) < 0.3] = -2000
    bounds = [(r * 7 // world, (r + 1) * 7 // world) for r in range(world)]
    wins = []
    for z0, z1 in bounds:
        nb = vol[z0:z1][vol[z0:z1] != -2000]
        wins.append([int(nb.min()), int(nb.max())] if nb.size else [2**31 - 1, -2**31])
    wins[-1] = [2**31 - 1, -2**31]  # pretend the last slab is all background
    _, lo, hi = oracle.preprocess(vol[: bounds[-1][0]])
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    port = _free_port()
    ps = [ctx.Process(target=_win_worker, args=(r, world, port, wins, ret)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(60)
    for r in range(world):
        assert ret[r] == [lo, hi]
