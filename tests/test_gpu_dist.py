"""Tuple-sharded multi-rank path on one GPU (-m gpu): two ranks (gloo
process group, both on cuda:0 -- NCCL refuses two ranks per device) must give
bit-identical per-slice results to the single-GPU tsa_segment."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_name, nz, z_first, k, units, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import phantom
    from paper_2012_10684_b200.dist import segment_tuple_sharded, slab_range

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg = phantom.CONFIGS[cfg_name]
        vol = phantom.make_volume(cfg, nz=nz, z_first=z_first)
        z0, z1 = slab_range(nz, world, rank)
        slab = torch.from_numpy(np.ascontiguousarray(vol[z0:z1])).cuda()
        out = segment_tuple_sharded(slab, nz, cfg.bins, k, cfg.qs[0], units=units)
        torch.cuda.synchronize()
        ret[rank] = (out["thresholds"].cpu().numpy(), out["objective"].cpu().numpy(),
                     out["status"].cpu().numpy(), out["labels"].cpu().numpy(), (z0, z1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k,units", [(4, 6), (3, 5), (2, 3)])
def test_tuple_sharded_equals_single_gpu(k, units):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import phantom
    import paper_2012_10684_b200 as tsa

    cfg = phantom.CONFIGS["c4"]
    nz, z_first = 5, 130
    vol = phantom.make_volume(cfg, nz=nz, z_first=z_first)
    ref = tsa.tsa_segment(torch.from_numpy(vol).cuda(), cfg.bins, k, cfg.qs[0], pipeline="staged",
                          units=units)
    torch.cuda.synchronize()
    mgr = mp.Manager()
    ret = mgr.dict()
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, "c4", nz, z_first, k, units, ret))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    for r in range(2):
        thr, phi, st, lab, (z0, z1) = ret[r]
        np.testing.assert_array_equal(thr, ref["thresholds"].cpu().numpy())
        np.testing.assert_array_equal(phi.view(np.int64), ref["objective"].cpu().numpy().view(np.int64))
        np.testing.assert_array_equal(st, ref["status"].cpu().numpy())
        np.testing.assert_array_equal(lab, ref["labels"].cpu().numpy()[z0:z1])
