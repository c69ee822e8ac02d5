"""The stream pipeline (k_stream.cuh: k_st_io + k_st_search, co-resident,
per-slice flags; the default for k = 2 above 1024 bins) against the staged
kernels (-m gpu): bit-identical histograms, thresholds, objective, status and
labels, on phantom slabs, degenerate slices, every objective mode and the
schedule knobs; plus the oracle on a c5 slab."""
import numpy as np
import pytest
import torch

import oracle
import phantom
import paper_2012_10684_b200 as tsa

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def same(a, b, what=""):
    for key in ("histogram", "thresholds", "status", "labels"):
        if a.get(key) is None and b.get(key) is None:
            continue
        assert torch.equal(a[key], b[key]), (what, key)
    if a.get("objective") is not None:
        assert torch.equal(a["objective"].view(torch.int64), b["objective"].view(torch.int64)), what


@pytest.mark.parametrize("q", [0.5, 0.8, 1.0, 1.3, 2.5])
def test_stream_equals_staged_c5_slab(q):
    cfg = phantom.CONFIGS["c5"]
    vol = torch.from_numpy(phantom.make_volume(cfg, nz=24, z_first=380)).to(DEV)
    p = tsa.make_problem(vol, cfg.bins, 2, q, pipeline="stream")
    assert tsa.tsa_pipeline_kind(p) == 3
    a = tsa.tsa_segment(vol, cfg.bins, 2, q, pipeline="stream")
    b = tsa.tsa_segment(vol, cfg.bins, 2, q, pipeline="staged")
    torch.cuda.synchronize()
    same(a, b, q)


@pytest.mark.parametrize("hc,lag", [(1, 1), (3, 2), (8, 8), (16, 30)])
def test_stream_schedule_invariance(hc, lag):
    cfg = phantom.CONFIGS["c5"]
    vol = torch.from_numpy(phantom.make_volume(cfg, nz=20, z_first=100)).to(DEV)
    ref = tsa.tsa_segment(vol, cfg.bins, 2, 0.8, pipeline="staged")
    out = tsa.tsa_segment(vol, cfg.bins, 2, 0.8, pipeline="stream", slab_slices=hc, label_lag=lag)
    torch.cuda.synchronize()
    same(out, ref, (hc, lag))


def test_stream_u8_and_degenerate_slices():
    """u8 input (forced stream), constant / two-level / overflow slices."""
    cfg = phantom.CONFIGS["c2"]
    v8 = phantom.make_volume(cfg, nz=10, z_first=140).copy()
    v8[2] = 9                       # constant: NO_VALID_SPLIT
    v8[4] = 0
    v8[4, :5] = 200                 # two levels: NO_VALID_SPLIT at k = 2
    v8[6, :3] = 254                 # fine at 256 bins
    for bins in (256, 255):         # 255 bins: the 254s are fine, 255s would overflow
        vv = v8.copy()
        if bins == 255:
            vv[7, 0, 0] = 255       # LEVEL_OVERFLOW
        vol = torch.from_numpy(vv).to(DEV)
        a = tsa.tsa_segment(vol, bins, 2, 0.8, pipeline="stream")
        b = tsa.tsa_segment(vol, bins, 2, 0.8, pipeline="staged")
        torch.cuda.synchronize()
        same(a, b, bins)
        st = a["status"].cpu().numpy()
        assert st[2] == 3 and st[4] == 3
        if bins == 255:
            assert st[7] == 2


def test_stream_optional_outputs():
    cfg = phantom.CONFIGS["c5"]
    vol = torch.from_numpy(phantom.make_volume(cfg, nz=9, z_first=700)).to(DEV)
    ref = tsa.tsa_segment(vol, cfg.bins, 2, 0.8, pipeline="staged")
    nz = vol.shape[0]
    for lab, obj in ((False, True), (True, False), (False, False)):
        out = {"thresholds": torch.empty((nz, 2), dtype=torch.int32, device=DEV),
               "objective": torch.empty(nz, dtype=torch.float64, device=DEV) if obj else None,
               "histogram": None, "status": torch.empty(nz, dtype=torch.int32, device=DEV),
               "labels": torch.empty(vol.shape, dtype=torch.uint8, device=DEV) if lab else None}
        tsa.tsa_segment(vol, cfg.bins, 2, 0.8, out=out, pipeline="stream")
        torch.cuda.synchronize()
        assert torch.equal(out["thresholds"], ref["thresholds"])
        assert torch.equal(out["status"], ref["status"])
        if lab:
            assert torch.equal(out["labels"], ref["labels"])
        if obj:
            assert torch.equal(out["objective"].view(torch.int64), ref["objective"].view(torch.int64))


def test_stream_repeated_calls_and_graph():
    """Workspace reuse across calls (counters re-zeroed) and CUDA-graph replay."""
    cfg = phantom.CONFIGS["c5"]
    vol = torch.from_numpy(phantom.make_volume(cfg, nz=12, z_first=300)).to(DEV)
    p = tsa.make_problem(vol, cfg.bins, 2, 0.8, pipeline="stream")
    ws = tsa.workspace_for(p, DEV)
    ref = tsa.tsa_segment(vol, cfg.bins, 2, 0.8, pipeline="staged")
    for _ in range(3):
        out = tsa.tsa_segment(vol, cfg.bins, 2, 0.8, workspace=ws, pipeline="stream")
        torch.cuda.synchronize()
        same(out, ref, "repeat")
    outg = {k: torch.empty_like(v) for k, v in ref.items()}
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tsa.tsa_segment(vol, cfg.bins, 2, 0.8, out=outg, workspace=ws, pipeline="stream")
    for _ in range(2):
        g.replay()
        torch.cuda.synchronize()
        same(outg, ref, "graph")


def test_stream_c5_slab_vs_oracle():
    cfg = phantom.CONFIGS["c5"]
    vh = phantom.make_volume(cfg, nz=6, z_first=450)
    out = tsa.tsa_segment(torch.from_numpy(vh).to(DEV), cfg.bins, 2, 0.8, pipeline="stream")
    torch.cuda.synchronize()
    ref = oracle.segment(vh, cfg.bins, 2, 0.8)
    np.testing.assert_array_equal(out["histogram"].cpu().numpy().astype(np.uint32), ref["hist"])
    thr = out["thresholds"].cpu().numpy()
    for z in range(vh.shape[0]):
        if tuple(thr[z]) != tuple(ref["thresholds"][z]):
            assert ref["gap"][z] < 1e-12
        else:
            np.testing.assert_array_equal(out["labels"][z].cpu().numpy(), ref["labels"][z])
    np.testing.assert_allclose(out["objective"].cpu().numpy(), ref["phi"], rtol=1e-12)
