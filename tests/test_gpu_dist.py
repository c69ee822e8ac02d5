"""Multi-rank paths on one GPU (-m gpu), through the C ABI.

tsa_segment_sharded (SURVEY.md §8(b),(e); "job distribution ...
reduction of results from different devices"):
* TUPLES with 2 and 3 ranks (gloo process group, the library's custom
  all-gather transport; all ranks on cuda:0 -- NCCL refuses two ranks per
  device) must give bit-identical per-slice results to the single-GPU
  tsa_segment, including a rank that owns no slice;
* the same with a 1-rank NCCL communicator (tsa_comm_init: NCCL inside
  libtsa);
* SLICES mode is tsa_segment of the slab;
* the in-library exchange equals the Python-driven one (dist.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_name, nz, z_first, k, units, enumeration, impl, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys

    sys.path.insert(0, ROOT)
    import phantom
    from paper_2012_10684_b200 import dist as tdist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg = phantom.CONFIGS[cfg_name]
        vol = phantom.make_volume(cfg, nz=nz, z_first=z_first)
        z0, z1 = tdist.slab_range(nz, world, rank)
        slab = torch.from_numpy(np.ascontiguousarray(vol[z0:z1])).cuda()
        fn = tdist.segment_tuple_sharded if impl == "lib" else tdist.segment_tuple_sharded_py
        out = fn(slab, nz, cfg.bins, k, cfg.qs[0], units=units, enumeration=enumeration)
        torch.cuda.synchronize()
        lab = out["labels"].cpu().numpy() if out["labels"] is not None else np.zeros((0,) + vol.shape[1:], np.uint8)
        ret[rank] = (out["thresholds"].cpu().numpy(), out["objective"].cpu().numpy(),
                     out["status"].cpu().numpy(), lab, (z0, z1), out["histogram"].cpu().numpy())
    finally:
        dist.destroy_process_group()


def _run(world, nz, z_first, k, units, enumeration="canonical", impl="lib"):
    mgr = mp.Manager()
    ret = mgr.dict()
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, "c4", nz, z_first, k, units, enumeration, impl, ret))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    return dict(ret)


def _reference(nz, z_first, k, units, enumeration="canonical"):
    import phantom
    import paper_2012_10684_b200 as tsa

    cfg = phantom.CONFIGS["c4"]
    vol = phantom.make_volume(cfg, nz=nz, z_first=z_first)
    ref = tsa.tsa_segment(torch.from_numpy(vol).cuda(), cfg.bins, k, cfg.qs[0], pipeline="staged",
                          units=units, enumeration=enumeration)
    torch.cuda.synchronize()
    return {key: v.cpu().numpy() for key, v in ref.items()}


def _check(ret, ref, world):
    for r in range(world):
        thr, phi, st, lab, (z0, z1), hist = ret[r]
        np.testing.assert_array_equal(thr, ref["thresholds"])
        np.testing.assert_array_equal(phi.view(np.int64), ref["objective"].view(np.int64))
        np.testing.assert_array_equal(st, ref["status"])
        np.testing.assert_array_equal(hist, ref["histogram"])
        np.testing.assert_array_equal(lab, ref["labels"][z0:z1])


@pytest.mark.parametrize("k,units,enumeration", [(4, 6, "canonical"), (3, 5, "canonical"),
                                                 (2, 3, "canonical"), (4, 0, "canonical"),
                                                 (4, 0, "dp"), (3, 0, "full")])
def test_tuple_sharded_c_abi_equals_single_gpu(k, units, enumeration):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    nz, z_first = 5, 130
    ref = _reference(nz, z_first, k, units, enumeration)
    _check(_run(2, nz, z_first, k, units, enumeration), ref, 2)


def test_tuple_sharded_rank_without_slices():
    """3 ranks over 2 slices: rank 2 owns no slice but still searches its units."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    ref = _reference(2, 200, 4, 7)
    _check(_run(3, 2, 200, 4, 7), ref, 3)


def test_library_exchange_equals_python_exchange():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    a = _run(2, 4, 60, 3, 4, impl="lib")
    b = _run(2, 4, 60, 3, 4, impl="py")
    for r in range(2):
        for x, y in zip(a[r][:4], b[r][:4]):
            np.testing.assert_array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


def test_nccl_comm_inside_library_single_rank():
    """tsa_comm_init over NCCL (one rank: the all-gathers are NCCL copies),
    then the tuple-sharded call: equal to tsa_segment bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import phantom
    import paper_2012_10684_b200 as tsa

    cfg = phantom.CONFIGS["c4"]
    vol = torch.from_numpy(phantom.make_volume(cfg, nz=6, z_first=100)).cuda()
    comm = tsa.TsaComm.nccl(1, 0, tsa.tsa_comm_unique_id())
    assert comm.kind == 1
    out = tsa.tsa_segment_sharded(vol, 6, cfg.bins, 4, 0.8, comm, mode="tuples", units=5)
    ref = tsa.tsa_segment(vol, cfg.bins, 4, 0.8, pipeline="staged", units=5)
    torch.cuda.synchronize()
    for key in ("thresholds", "status", "histogram", "labels"):
        assert torch.equal(out[key], ref[key]), key
    assert torch.equal(out["objective"].view(torch.int64), ref["objective"].view(torch.int64))
    sl = tsa.tsa_segment_sharded(vol, 6, cfg.bins, 4, 0.8, comm, mode="slices")
    torch.cuda.synchronize()
    for key in ("thresholds", "status", "histogram", "labels"):
        assert torch.equal(sl[key], ref[key]), key
    comm.close()
