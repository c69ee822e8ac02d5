"""The overlap pipeline (tsa_segment pipeline = 4: staged kernels on slabs over
two streams; opt-in: measured slower than the staged kernels on c5) against
the staged kernels, bit for bit (-m gpu)."""
import pytest
import torch

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


@pytest.mark.parametrize("q", [0.5, 0.8, 1.0, 1.7])
@pytest.mark.parametrize("nz,slabs", [(40, 0), (17, 3), (9, 64)])
def test_overlap_equals_staged_c5(q, nz, slabs):
    cfg = phantom.CONFIGS["c5"]
    vol = torch.from_numpy(phantom.make_volume(cfg, nz=nz, z_first=200)).to(DEV)
    assert tsa.tsa_pipeline_kind(tsa.make_problem(vol, cfg.bins, 2, q, pipeline="overlap")) == 4
    a = tsa.tsa_segment(vol, cfg.bins, 2, q, pipeline="overlap", slab_slices=slabs)
    b = tsa.tsa_segment(vol, cfg.bins, 2, q, pipeline="staged")
    torch.cuda.synchronize()
    same(a, b, (q, nz, slabs))


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_overlap_any_problem(k):
    cfg = phantom.CONFIGS["c2"]
    v8 = phantom.make_volume(cfg, nz=21, z_first=100).copy()
    v8[4] = 3  # NO_VALID_SPLIT slice
    vol = torch.from_numpy(v8).to(DEV)
    a = tsa.tsa_segment(vol, 256, k, 0.8, pipeline="overlap", slab_slices=5)
    b = tsa.tsa_segment(vol, 256, k, 0.8, pipeline="staged")
    torch.cuda.synchronize()
    same(a, b, k)


def test_overlap_optional_outputs_and_capture():
    cfg = phantom.CONFIGS["c5"]
    vol = torch.from_numpy(phantom.make_volume(cfg, nz=20, z_first=600)).to(DEV)
    ref = tsa.tsa_segment(vol, cfg.bins, 2, 0.8, pipeline="staged")
    nz = vol.shape[0]
    out = {"thresholds": torch.empty((nz, 2), dtype=torch.int32, device=DEV), "objective": None,
           "histogram": None, "status": None, "labels": None}
    tsa.tsa_segment(vol, cfg.bins, 2, 0.8, out=out, pipeline="overlap")
    torch.cuda.synchronize()
    assert torch.equal(out["thresholds"], ref["thresholds"])
    # inside a CUDA-graph capture the call runs the staged kernels on one stream
    p = tsa.make_problem(vol, cfg.bins, 2, 0.8)
    ws = tsa.workspace_for(p, DEV)
    outg = {kk: torch.empty_like(v) for kk, v in ref.items()}
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tsa.tsa_segment(vol, cfg.bins, 2, 0.8, out=outg, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    same(outg, ref, "graph")
