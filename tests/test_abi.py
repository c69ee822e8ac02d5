"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/tsa.h declares, validates arguments synchronously and sizes
workspaces.  (No compute calls: there is no device here.)"""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2012_10684_b200 as tsa
from paper_2012_10684_b200 import tsa_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "tsa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsa(?:2d)?_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(tsa.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build_tsa()
    return tsa.load()


def test_exports_every_declared_symbol(lib):
    declared = header_functions()
    assert set(declared) == set(tsa.EXPORTS), declared
    out = subprocess.check_output(["nm", "-D", "--defined-only", tsa.LIB_PATH]).decode()
    exported = set(re.findall(r"\bT (tsa(?:2d)?_[a-z_0-9]+)", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    for f in declared:
        assert hasattr(lib, f)


def test_sm100a_cubin_embedded(lib):
    out = subprocess.check_output(["cuobjdump", "--list-elf", tsa.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_version_and_strings(lib):
    assert tsa.tsa_version() == 1
    assert lib.tsa_status_string(3) == b"TSA_ERR_NO_VALID_SPLIT"


def _p(**kw):
    base = dict(volume=256, dtype=1, nx=512, ny=512, nz=300, bins=256, k=2, q=0.8, objective=0,
                enumeration=0, units_per_slice=0)
    base.update(kw)
    return tsa_problem(**base)


@pytest.mark.parametrize(
    "kw",
    [dict(q=0.0), dict(q=-1.0), dict(q=float("inf")), dict(q=float("nan")), dict(k=0), dict(k=5),
     dict(bins=1), dict(bins=4097, dtype=2), dict(bins=300, dtype=1), dict(nx=0), dict(nz=-1),
     dict(k=3, bins=3), dict(volume=0), dict(dtype=3), dict(objective=2), dict(enumeration=7),
     dict(nx=65536, ny=65536), dict(nz=65536)],
)
def test_invalid_arguments_rejected_synchronously(lib, kw):
    p = _p(**kw)
    assert lib.tsa_validate(ctypes.byref(p)) == tsa.TSA_ERR_INVALID_ARG
    assert lib.tsa_workspace_size(ctypes.byref(p)) == 0
    # entry points return the error before touching the device
    o = tsa.tsa_outputs(1, 0, 0, 0, 0)
    assert lib.tsa_segment(ctypes.byref(p), ctypes.byref(o), ctypes.c_void_p(1), 1 << 40, None) == 1
    assert lib.tsa_histogram(ctypes.byref(p), ctypes.c_void_p(1), ctypes.c_void_p(1), None) == 1
    assert lib.tsa_label(ctypes.byref(p), ctypes.c_void_p(1), None, ctypes.c_void_p(1), None) == 1
    assert len(lib.tsa_last_error()) > 0


def test_pipeline_kind(lib):
    assert lib.tsa_pipeline_kind(ctypes.byref(_p())) == 2            # c2: compact
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(pipeline=1))) == 1  # persistent fused
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(k=3))) == -1        # k >= 3: staged
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(pipeline=-1))) == -1
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(enumeration=1))) == -1
    # k = 2 above 1024 bins (c5): the stream pipeline; forced stream on an eligible u8 problem
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(dtype=2, bins=4096, nx=1024, ny=1024))) in (4, -1)
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(dtype=2, bins=4096, nx=1024, ny=1024, nz=8))) == -1
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(k=3, pipeline=4))) == 4
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(pipeline=3))) == 3
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(pipeline=3, k=3))) == -1
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(dtype=2, bins=4096, nx=1024, ny=1024, k=1))) == -1
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(nx=37, ny=53))) == -1  # n % 16 != 0
    assert lib.tsa_pipeline_kind(ctypes.byref(_p(q=0.0))) == 0


def test_valid_problems_and_workspace(lib):
    for kw in (dict(), dict(k=4), dict(k=1, nx=256, ny=256, nz=1), dict(dtype=2, bins=4096, nx=1024,
               ny=1024, nz=1000), dict(q=1.0), dict(objective=1, k=3), dict(enumeration=1, k=4)):
        p = _p(**kw)
        assert lib.tsa_validate(ctypes.byref(p)) == 0, kw
        ws = lib.tsa_workspace_size(ctypes.byref(p))
        assert ws > 0 and ws % 256 == 0
    # a too-small workspace is reported, not overrun
    p = _p()
    o = tsa.tsa_outputs(1, 0, 0, 0, 0)
    assert lib.tsa_segment(ctypes.byref(p), ctypes.byref(o), ctypes.c_void_p(256), 10, None) == \
        tsa.TSA_ERR_WORKSPACE


def test_search_argument_checks(lib):
    ws = lib.tsa_search_workspace_size(300, 512 * 512, 256, 2, 0.8, 0, 0)
    assert ws > 0
    assert lib.tsa_search_workspace_size(300, 512 * 512, 256, 5, 0.8, 0, 0) == 0
    one = ctypes.c_void_p(1)
    # bad unit range
    assert lib.tsa_search(one, one, 300, 512 * 512, 256, 2, 0.8, 0, 0, 8, 4, 9, one, one, one, ws,
                          None) == tsa.TSA_ERR_INVALID_ARG
    # too-small workspace
    assert lib.tsa_search(one, one, 300, 512 * 512, 256, 2, 0.8, 0, 0, 8, 0, 8, one, one, one, 16,
                          None) == tsa.TSA_ERR_WORKSPACE
    assert lib.tsa_default_units(300, 256, 2, 0) >= 1
    assert lib.tsa_default_units(300, 256, 4, 0) >= lib.tsa_default_units(300, 256, 2, 0)


def test_compute_calls_refuse_cpu_tensors():
    import torch

    vol = torch.zeros((1, 16, 16), dtype=torch.uint8)
    with pytest.raises(ValueError):
        tsa.tsa_segment(vol, 256, 1, 0.8)


def test_key_unpack():
    assert tsa.unpack_key((3 << 36) | (70 << 24) | (71 << 12) | 254, 4) == (3, 70, 71, 254)


# ------------------------------------------------ §8(f) entry points (no GPU)
def _p2(**kw):
    base = dict(volume=16, nx=512, ny=512, nz=300, bins=256, q=0.8, cluster=0)
    base.update(kw)
    return tsa.tsa2d_problem(**base)


@pytest.mark.parametrize("kw", [dict(bins=1), dict(bins=257), dict(q=0.0), dict(q=float("nan")),
                                dict(nx=0), dict(nx=70000, ny=1), dict(volume=0), dict(cluster=3),
                                dict(cluster=9)])
def test_2d_invalid_arguments(lib, kw):
    p = _p2(**kw)
    assert lib.tsa2d_validate(ctypes.byref(p)) == tsa.TSA_ERR_INVALID_ARG
    assert lib.tsa2d_workspace_size(ctypes.byref(p)) == 0
    o = tsa.tsa_outputs(1, 0, 0, 0, 0)
    assert lib.tsa2d_segment(ctypes.byref(p), ctypes.byref(o), ctypes.c_void_p(1), 1 << 40, None) == 1
    assert lib.tsa2d_mean3x3(ctypes.byref(p), ctypes.c_void_p(1), None) == 1


def test_2d_plan(lib):
    """Cluster size: the smallest in 4..8 whose CTAs count <= 65536 pixels (one
    held out) and whose shared-memory plan fits (4 for a 512x512 slice)."""
    assert lib.tsa2d_cluster_size(ctypes.byref(_p2())) == 4
    assert lib.tsa2d_cluster_size(ctypes.byref(_p2(ny=513))) == 5
    assert lib.tsa2d_cluster_size(ctypes.byref(_p2(bins=64, nx=64, ny=64))) == 4
    assert lib.tsa2d_cluster_size(ctypes.byref(_p2(nx=1024, ny=1024))) == 8  # several rounds
    assert lib.tsa2d_workspace_size(ctypes.byref(_p2())) > 0


def _ph(**kw):
    base = dict(volume=16, nx=512, ny=512, nz=300, background=-2000, k=2, q=0.8, objective=0,
                enumeration=0)
    base.update(kw)
    return tsa.tsa_hu_problem(**base)


@pytest.mark.parametrize("kw", [dict(volume=8), dict(nx=7, ny=7), dict(k=5), dict(q=-1.0),
                                dict(background=5000), dict(objective=3), dict(volume=0)])
def test_hu_invalid_arguments(lib, kw):
    p = _ph(**kw)
    assert lib.tsa_hu_workspace_size(ctypes.byref(p)) == 0
    o = tsa.tsa_outputs(1, 0, 0, 0, 0)
    one = ctypes.c_void_p(256)
    assert lib.tsa_hu_segment(ctypes.byref(p), ctypes.byref(o), None, one, 1 << 40, None) == 1
    assert lib.tsa_hu_preprocess(ctypes.byref(p), one, None, one, 1 << 40, None) == 1
    assert lib.tsa_hu_histogram(ctypes.byref(p), one, one, 1 << 40, None) == 1


def test_hu_workspace_and_dp_rules(lib):
    assert lib.tsa_hu_workspace_size(ctypes.byref(_ph())) > 0
    # the DP needs the pseudo-additive objective and one work unit per slice
    assert lib.tsa_validate(ctypes.byref(_p(enumeration=2, k=4))) == 0
    assert lib.tsa_validate(ctypes.byref(_p(enumeration=2, objective=1))) == tsa.TSA_ERR_INVALID_ARG
    assert lib.tsa_default_units(300, 256, 4, 2) == 1


@pytest.mark.parametrize("args", [(0, 1, 8, 8, 1, 10, 3), (16, 16, 8, 8, 1, 10, 3),
                                  (16, 32, 8, 8, 1, 11, 3), (16, 32, 8, 8, 1, 10, 4),
                                  (16, 32, 0, 8, 1, 10, 0), (16, 32, 8, 8, 1, -1, 0)])
def test_morph_invalid_arguments(lib, args):
    inp, out, nx, ny, nz, r, op = args
    assert lib.tsa_morph(ctypes.c_void_p(inp) if inp else None, ctypes.c_void_p(out), nx, ny, nz, r,
                         op, None, 0, None) == tsa.TSA_ERR_INVALID_ARG


def test_morph_workspace(lib):
    assert lib.tsa_morph_workspace_size(512, 512, 300, 3) >= 512 * 512 * 300
    assert lib.tsa_morph_workspace_size(512, 512, 300, 0) == 0
    # OPEN / TOPHAT without workspace: reported, nothing launched
    assert lib.tsa_morph(ctypes.c_void_p(16), ctypes.c_void_p(32), 8, 8, 1, 3, 2, None, 0, None) == \
        tsa.TSA_ERR_WORKSPACE


# ------------------------------------------------------ q sweep / multi-GPU ABI
def test_sweep_workspace_and_validation(lib):
    p = _p(k=3, bins=256, nz=600)
    qs = (ctypes.c_double * 11)(*[0.5 + 0.1 * i for i in range(11)])
    n = lib.tsa_sweep_workspace_size(ctypes.byref(p), qs, 11)
    assert n >= lib.tsa_workspace_size(ctypes.byref(p))
    bad = (ctypes.c_double * 2)(0.8, 0.0)
    assert lib.tsa_sweep_workspace_size(ctypes.byref(p), bad, 2) == 0
    assert lib.tsa_sweep_workspace_size(ctypes.byref(p), qs, 0) == 0
    o = (tsa.tsa_outputs * 2)(tsa.tsa_outputs(1, 0, 0, 0, 0), tsa.tsa_outputs(1, 0, 0, 0, 0))
    assert lib.tsa_segment_sweep(ctypes.byref(p), bad, 2, o, ctypes.c_void_p(1), 1 << 40, None) == 1


@pytest.mark.parametrize("nz,world", [(1, 1), (7, 3), (300, 8), (301, 8), (2, 3), (1000, 7)])
def test_slab_range_matches_python_partition(lib, nz, world):
    from paper_2012_10684_b200.dist import slab_range

    for r in range(world):
        assert tsa.tsa_slab_range(nz, world, r) == slab_range(nz, world, r)


def test_sharded_units_are_rank_independent(lib):
    """The tuple-sharded unit count never depends on the local device
    (mixed SM counts must not split the unit space differently)."""
    for k, bins, enum in ((4, 256, 0), (3, 256, 0), (2, 4096, 0), (4, 256, 1)):
        p = _p(k=k, bins=bins, enumeration=enum, dtype=1 if bins <= 256 else 2, nz=38)
        u = {lib.tsa_sharded_units(ctypes.byref(p), 300, P) for P in (8,)}
        assert len(u) == 1 and min(u) >= 8
    p = _p(k=4, enumeration=2)
    assert lib.tsa_sharded_units(ctypes.byref(p), 300, 8) == 1  # DP: one unit per slice


def test_custom_comm_lifecycle_and_errors(lib):
    calls = []
    comm = tsa.TsaComm.custom(2, 1, lambda *a: calls.append(a))
    assert comm.kind == 2
    p = _p(k=4, nz=150)
    assert lib.tsa_sharded_workspace_size(ctypes.byref(p), 300, 1, comm.handle) > 0
    assert lib.tsa_sharded_workspace_size(ctypes.byref(p), 300, 0, comm.handle) == \
        lib.tsa_workspace_size(ctypes.byref(p))
    o = tsa.tsa_outputs(1, 0, 0, 0, 0)
    # wrong slab size for rank 1 of 2 over 301 slices (150 expected), bad mode
    bad = _p(k=4, nz=151)
    assert lib.tsa_segment_sharded(ctypes.byref(bad), 301, ctypes.byref(o), 1, comm.handle,
                                   ctypes.c_void_p(1), 1 << 40, None) == 1
    assert lib.tsa_segment_sharded(ctypes.byref(p), 300, ctypes.byref(o), 7, comm.handle,
                                   ctypes.c_void_p(1), 1 << 40, None) == 1
    assert lib.tsa_segment_sharded(ctypes.byref(p), 300, ctypes.byref(o), 1, None,
                                   ctypes.c_void_p(1), 1 << 40, None) == 1
    assert not calls  # nothing was exchanged before the arguments were rejected
    comm.close()
    h = ctypes.c_void_p()
    assert lib.tsa_comm_init_custom(ctypes.byref(h), 2, 2, tsa.ALLGATHER_FN(lambda *a: 0), None) == 1
    assert lib.tsa_comm_init(ctypes.byref(h), 0, 0, ctypes.create_string_buffer(128)) == 1
