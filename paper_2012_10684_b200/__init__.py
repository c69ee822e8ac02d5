"""B200-native Tsallis multilevel thresholding (arXiv 2012.10684 hot path).

Thin Python binding over ``libtsa.so`` (C ABI in ``include/tsa.h``): argument
marshalling only -- every step of the path runs in the library's sm_100a CUDA
kernels.  PyTorch supplies device memory (tensors), streams
(``torch.cuda.current_stream()``) and, for multi-GPU runs, process groups.
There is no CPU fallback: importing works anywhere (so the ABI can be checked
on a CPU host) but every compute call requires CUDA tensors and the built
library, and raises otherwise.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# TSA_LIB_PATH: an alternative build of the same library (A/B experiments in tools/)
LIB_PATH = os.environ.get("TSA_LIB_PATH") or os.path.join(_HERE, "libtsa.so")

TSA_OK, TSA_ERR_INVALID_ARG, TSA_ERR_LEVEL_OVERFLOW, TSA_ERR_NO_VALID_SPLIT = 0, 1, 2, 3
TSA_ERR_WORKSPACE, TSA_ERR_CUDA, TSA_ERR_NCCL = 4, 5, 6
TSA_U8, TSA_U16 = 1, 2
TSA_OBJ_PSEUDO_ADDITIVE, TSA_OBJ_SUM_PLUS_PRODUCT = 0, 1
TSA_ENUM_CANONICAL, TSA_ENUM_FULL, TSA_ENUM_DP = 0, 1, 2
TSA_KEY_NONE = 0xFFFFFFFFFFFFFFFF
KMAX = 4

OBJECTIVES = {"pseudo_additive": 0, "sum_plus_product": 1}
ENUMERATIONS = {"canonical": 0, "full": 1, "dp": 2}

# every symbol include/tsa.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "tsa_validate", "tsa_workspace_size", "tsa_segment", "tsa_histogram",
    "tsa_search_workspace_size", "tsa_default_units", "tsa_search", "tsa_merge",
    "tsa_finalize", "tsa_label", "tsa_segment_host_scratch_size", "tsa_segment_host",
    "tsa_status_string", "tsa_last_error", "tsa_version", "tsa_pipeline_kind",
    "tsa2d_validate", "tsa2d_workspace_size", "tsa2d_cluster_size", "tsa2d_segment",
    "tsa2d_histogram", "tsa2d_mean3x3",
    "tsa_hu_workspace_size", "tsa_hu_segment", "tsa_hu_preprocess", "tsa_hu_histogram",
    "tsa_hu_finish",
    "tsa_morph_workspace_size", "tsa_morph",
    "tsa_class_consts_workspace_size", "tsa_class_consts",
    "tsa_sweep_workspace_size", "tsa_segment_sweep",
    "tsa_comm_unique_id", "tsa_comm_init", "tsa_comm_init_custom", "tsa_comm_destroy",
    "tsa_comm_kind", "tsa_slab_range", "tsa_sharded_units", "tsa_sharded_workspace_size",
    "tsa_segment_sharded",
)
TSA_SHARD_SLICES, TSA_SHARD_TUPLES = 0, 1
SHARD_MODES = {"slices": 0, "tuples": 1}
COMM_ID_BYTES = 128
# int (*)(void *user, const void *send, void *recv, size_t bytes, void *stream)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_size_t, ctypes.c_void_p)


class TsaError(RuntimeError):
    def __init__(self, status, where, detail=""):
        super().__init__(f"{where}: status {status} ({_status_name(status)}) {detail}")
        self.status = status


def _status_name(s):
    names = {0: "TSA_OK", 1: "TSA_ERR_INVALID_ARG", 2: "TSA_ERR_LEVEL_OVERFLOW",
             3: "TSA_ERR_NO_VALID_SPLIT", 4: "TSA_ERR_WORKSPACE", 5: "TSA_ERR_CUDA",
             6: "TSA_ERR_NCCL"}
    return names.get(int(s), "?")


class tsa_problem(ctypes.Structure):
    _fields_ = [
        ("volume", ctypes.c_void_p),
        ("dtype", ctypes.c_int32),
        ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
        ("bins", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("q", ctypes.c_double),
        ("objective", ctypes.c_int32),
        ("enumeration", ctypes.c_int32),
        ("units_per_slice", ctypes.c_int32),
        ("pipeline", ctypes.c_int32),
        ("slab_slices", ctypes.c_int32),
        ("label_lag", ctypes.c_int32),
    ]


class tsa_outputs(ctypes.Structure):
    _fields_ = [
        ("thresholds", ctypes.c_void_p),
        ("labels", ctypes.c_void_p),
        ("objective", ctypes.c_void_p),
        ("histogram", ctypes.c_void_p),
        ("slice_status", ctypes.c_void_p),
    ]


class tsa2d_problem(ctypes.Structure):
    _fields_ = [
        ("volume", ctypes.c_void_p),
        ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
        ("bins", ctypes.c_int32),
        ("q", ctypes.c_double),
        ("cluster", ctypes.c_int32),
    ]


class tsa_hu_problem(ctypes.Structure):
    _fields_ = [
        ("volume", ctypes.c_void_p),
        ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
        ("background", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("q", ctypes.c_double),
        ("objective", ctypes.c_int32),
        ("enumeration", ctypes.c_int32),
    ]


_lib = None


def library_path() -> str:
    return LIB_PATH


def load() -> ctypes.CDLL:
    """Load libtsa.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, D, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
    PP = ctypes.POINTER(tsa_problem)
    PO = ctypes.POINTER(tsa_outputs)
    P2 = ctypes.POINTER(tsa2d_problem)
    PH = ctypes.POINTER(tsa_hu_problem)
    sig = {
        "tsa_validate": (I32, [PP]),
        "tsa_workspace_size": (SZ, [PP]),
        "tsa_segment": (I32, [PP, PO, P, SZ, P]),
        "tsa_histogram": (I32, [PP, P, P, P]),
        "tsa_search_workspace_size": (SZ, [I64, I64, I32, I32, D, I32, I32]),
        "tsa_default_units": (I32, [I64, I32, I32, I32]),
        "tsa_search": (I32, [P, P, I64, I64, I32, I32, D, I32, I32, I32, I32, I32, P, P, P, SZ, P]),
        "tsa_merge": (I32, [P, P, I32, I64, P, P, P]),
        "tsa_finalize": (I32, [P, P, I64, I32, I32, D, I32, P, P, I32, PO, P]),
        "tsa_label": (I32, [PP, P, P, P, P]),
        "tsa_segment_host_scratch_size": (SZ, [PP, I64]),
        "tsa_segment_host": (I32, [PP, I64, P, P, P, P, P, SZ, P, P]),
        "tsa_status_string": (ctypes.c_char_p, [I32]),
        "tsa_last_error": (ctypes.c_char_p, []),
        "tsa_version": (I32, []),
        "tsa_pipeline_kind": (I32, [PP]),
        "tsa2d_validate": (I32, [P2]),
        "tsa2d_workspace_size": (SZ, [P2]),
        "tsa2d_cluster_size": (I32, [P2]),
        "tsa2d_segment": (I32, [P2, PO, P, SZ, P]),
        "tsa2d_histogram": (I32, [P2, P, P, P, SZ, P]),
        "tsa2d_mean3x3": (I32, [P2, P, P]),
        "tsa_hu_workspace_size": (SZ, [PH]),
        "tsa_hu_segment": (I32, [PH, PO, P, P, SZ, P]),
        "tsa_hu_preprocess": (I32, [PH, P, P, P, SZ, P]),
        "tsa_hu_histogram": (I32, [PH, P, P, SZ, P]),
        "tsa_hu_finish": (I32, [PH, P, PO, P, SZ, P]),
        "tsa_morph_workspace_size": (SZ, [I64, I64, I64, I32]),
        "tsa_morph": (I32, [P, P, I64, I64, I64, I32, I32, P, SZ, P]),
        "tsa_class_consts_workspace_size": (SZ, []),
        "tsa_class_consts": (I32, [P, I64, D, P, P, P, SZ, P]),
        "tsa_sweep_workspace_size": (SZ, [PP, P, I32]),
        "tsa_segment_sweep": (I32, [PP, P, I32, PO, P, SZ, P]),
        "tsa_comm_unique_id": (I32, [P]),
        "tsa_comm_init": (I32, [ctypes.POINTER(P), I32, I32, P]),
        "tsa_comm_init_custom": (I32, [ctypes.POINTER(P), I32, I32, ALLGATHER_FN, P]),
        "tsa_comm_destroy": (I32, [P]),
        "tsa_comm_kind": (I32, [P]),
        "tsa_slab_range": (I32, [I64, I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "tsa_sharded_units": (I32, [PP, I64, I32]),
        "tsa_sharded_workspace_size": (SZ, [PP, I64, I32, P]),
        "tsa_segment_sharded": (I32, [PP, I64, PO, I32, P, P, SZ, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(status, where):
    if status != TSA_OK:
        detail = load().tsa_last_error().decode(errors="replace")
        raise TsaError(status, where, detail)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libtsa needs CUDA tensors (no CPU fallback)")


def _dtype_code(vol):
    if vol.dtype == torch.uint8:
        return TSA_U8
    if vol.dtype == torch.uint16:
        return TSA_U16
    raise ValueError(f"volume dtype must be uint8 or uint16, got {vol.dtype}")


PIPELINES = {"auto": 0, "fused": 1, "compact": 2, "staged": -1, "stream": 3, "overlap": 4}


def make_problem(vol, bins, k, q, objective="pseudo_additive", enumeration="canonical", units=0,
                 pipeline="auto", slab_slices=0, label_lag=0):
    if vol.dim() != 3 or not vol.is_contiguous():
        raise ValueError("volume must be a contiguous [nz][ny][nx] tensor")
    nz, ny, nx = vol.shape
    return tsa_problem(vol.data_ptr(), _dtype_code(vol), nx, ny, nz, bins, k, float(q),
                       OBJECTIVES.get(objective, objective), ENUMERATIONS.get(enumeration, enumeration),
                       units, PIPELINES.get(pipeline, pipeline), slab_slices, label_lag)


def tsa_version():
    return int(load().tsa_version())


def tsa_validate(problem):
    return int(load().tsa_validate(ctypes.byref(problem)))


def tsa_pipeline_kind(problem):
    """2 = compact (3 kernels), 1 = fused persistent kernel, -1 = staged kernels, 0 = invalid."""
    return int(load().tsa_pipeline_kind(ctypes.byref(problem)))


def tsa_workspace_size(problem):
    return int(load().tsa_workspace_size(ctypes.byref(problem)))


def tsa_default_units(nz, bins, k, enumeration="canonical"):
    return int(load().tsa_default_units(nz, bins, k, ENUMERATIONS.get(enumeration, enumeration)))


def tsa_search_workspace_size(nz, voxels_per_slice, bins, k, q, objective="pseudo_additive",
                              enumeration="canonical"):
    return int(load().tsa_search_workspace_size(nz, voxels_per_slice, bins, k, float(q),
                                                OBJECTIVES.get(objective, objective),
                                                ENUMERATIONS.get(enumeration, enumeration)))


def workspace_for(problem, device):
    n = tsa_workspace_size(problem)
    if n == 0:
        _check(load().tsa_validate(ctypes.byref(problem)), "tsa_workspace_size")
    return torch.empty(n, dtype=torch.uint8, device=device)


def tsa_segment(vol, bins, k, q, objective="pseudo_additive", enumeration="canonical", units=0,
                labels=True, out=None, workspace=None, stream=None, pipeline="auto", slab_slices=0,
                label_lag=0):
    """Whole path on the current stream.  Returns dict of device tensors:
    thresholds [nz,k] i32, objective [nz] f64, histogram [nz,bins] u32,
    status [nz] i32, labels [nz,ny,nx] u8 (or None)."""
    _need_cuda(vol)
    lib = load()
    p = make_problem(vol, bins, k, q, objective, enumeration, units, pipeline, slab_slices, label_lag)
    nz = vol.shape[0]
    dev = vol.device
    if out is None:
        out = {
            "thresholds": torch.empty((nz, k), dtype=torch.int32, device=dev),
            "objective": torch.empty(nz, dtype=torch.float64, device=dev),
            "histogram": torch.empty((nz, bins), dtype=torch.int32, device=dev),
            "status": torch.empty(nz, dtype=torch.int32, device=dev),
            "labels": torch.empty(vol.shape, dtype=torch.uint8, device=dev) if labels else None,
        }
    o = tsa_outputs(out["thresholds"].data_ptr(),
                    out["labels"].data_ptr() if out.get("labels") is not None else None,
                    out["objective"].data_ptr() if out.get("objective") is not None else None,
                    out["histogram"].data_ptr() if out.get("histogram") is not None else None,
                    out["status"].data_ptr() if out.get("status") is not None else None)
    if workspace is None:
        workspace = workspace_for(p, dev)
    _check(lib.tsa_segment(ctypes.byref(p), ctypes.byref(o), _ptr(workspace), workspace.numel(),
                           _stream(stream)), "tsa_segment")
    return out


def tsa_histogram(vol, bins, stream=None, out=None):
    """(hist [nz,bins] i32 (u32 bits), status [nz] i32); out = (hist, status) to reuse buffers."""
    _need_cuda(vol)
    p = make_problem(vol, bins, 1, 1.0)
    nz = vol.shape[0]
    if out is not None:
        hist, status = out
    else:
        hist = torch.empty((nz, bins), dtype=torch.int32, device=vol.device)
        status = torch.empty(nz, dtype=torch.int32, device=vol.device)
    _check(load().tsa_histogram(ctypes.byref(p), _ptr(hist), _ptr(status), _stream(stream)),
           "tsa_histogram")
    return hist, status


def tsa_search(hist, status, voxels_per_slice, k, q, objective="pseudo_additive",
               enumeration="canonical", units=0, unit_begin=0, unit_end=None, workspace=None,
               stream=None, out=None):
    """Returns (part_score [n_units, nz] f64, part_key [n_units, nz] i64 (u64 bits)).
    `status` is updated in place (NO_VALID_SPLIT)."""
    _need_cuda(hist, status)
    nz, bins = hist.shape
    obj = OBJECTIVES.get(objective, objective)
    enum = ENUMERATIONS.get(enumeration, enumeration)
    if units <= 0:
        units = tsa_default_units(nz, bins, k, enum)
    unit_end = units if unit_end is None else unit_end
    nu = unit_end - unit_begin
    if out is not None:
        ps, pk = out
    else:
        ps = torch.empty((max(nu, 1), nz), dtype=torch.float64, device=hist.device)
        pk = torch.empty((max(nu, 1), nz), dtype=torch.int64, device=hist.device)
    if workspace is None:
        n = tsa_search_workspace_size(nz, voxels_per_slice, bins, k, q, obj, enum)
        workspace = torch.empty(max(n, 1), dtype=torch.uint8, device=hist.device)
    _check(load().tsa_search(_ptr(hist), _ptr(status), nz, voxels_per_slice, bins, k, float(q), obj,
                             enum, units, unit_begin, unit_end, _ptr(ps), _ptr(pk),
                             _ptr(workspace), workspace.numel(), _stream(stream)), "tsa_search")
    return ps, pk


def tsa_merge(part_score, part_key, stream=None):
    _need_cuda(part_score, part_key)
    nparts, nz = part_score.shape
    s = torch.empty(nz, dtype=torch.float64, device=part_score.device)
    k = torch.empty(nz, dtype=torch.int64, device=part_score.device)
    _check(load().tsa_merge(_ptr(part_score), _ptr(part_key), nparts, nz, _ptr(s), _ptr(k),
                            _stream(stream)), "tsa_merge")
    return s, k


def tsa_finalize(hist, status, k, q, part_score, part_key, objective="pseudo_additive", stream=None,
                 out=None):
    _need_cuda(hist, status, part_score, part_key)
    nz, bins = hist.shape
    nparts = part_score.shape[0]
    dev = hist.device
    if out is not None:
        thr, phi, st = out
    else:
        thr = torch.empty((nz, k), dtype=torch.int32, device=dev)
        phi = torch.empty(nz, dtype=torch.float64, device=dev)
        st = torch.empty(nz, dtype=torch.int32, device=dev)
    o = tsa_outputs(thr.data_ptr(), None, phi.data_ptr(), None, st.data_ptr())
    _check(load().tsa_finalize(_ptr(hist), _ptr(status), nz, bins, k, float(q),
                               OBJECTIVES.get(objective, objective), _ptr(part_score),
                               _ptr(part_key), nparts, ctypes.byref(o), _stream(stream)),
           "tsa_finalize")
    return thr, phi, st


def tsa_label(vol, thresholds, status=None, bins=None, stream=None, out=None):
    _need_cuda(vol, thresholds, status)
    k = thresholds.shape[1]
    bins = bins or (256 if vol.dtype == torch.uint8 else 4096)
    p = make_problem(vol, bins, k, 1.0)
    labels = out if out is not None else torch.empty(vol.shape, dtype=torch.uint8, device=vol.device)
    _check(load().tsa_label(ctypes.byref(p), _ptr(thresholds), _ptr(status), _ptr(labels),
                            _stream(stream)), "tsa_label")
    return labels


def tsa_segment_host(vol_host, bins, k, q, objective="pseudo_additive", enumeration="canonical",
                     units=0, slab=None, labels=True, scratch=None, streams=None, out=None,
                     device=None, pipeline="auto"):
    """Host-buffer path: vol_host is a CPU (ideally pinned) torch tensor; copies
    in/out run inside the library, overlapped with compute on two streams.
    Returns dict of CPU tensors.  Blocks until done."""
    if vol_host.is_cuda:
        raise ValueError("tsa_segment_host takes a host tensor")
    device = device or torch.device("cuda", torch.cuda.current_device())
    lib = load()
    p = make_problem(vol_host, bins, k, q, objective, enumeration, units, pipeline)
    nz = vol_host.shape[0]
    slab = slab or max(1, min(nz, 50))  # measured best on c2 (tools/exp_e2e.py)
    if out is None:
        pin = vol_host.is_pinned()
        out = {
            "thresholds": torch.empty((nz, k), dtype=torch.int32, pin_memory=pin),
            "objective": torch.empty(nz, dtype=torch.float64, pin_memory=pin),
            "status": torch.empty(nz, dtype=torch.int32, pin_memory=pin),
            "labels": torch.empty(vol_host.shape, dtype=torch.uint8, pin_memory=pin) if labels else None,
        }
    if scratch is None:
        n = int(lib.tsa_segment_host_scratch_size(ctypes.byref(p), slab))
        scratch = torch.empty(max(n, 1), dtype=torch.uint8, device=device)
    if streams is None:
        streams = (torch.cuda.current_stream(device), torch.cuda.Stream(device))
    lab = out.get("labels")
    _check(lib.tsa_segment_host(ctypes.byref(p), slab, _ptr(out["thresholds"]), _ptr(out["objective"]),
                                _ptr(out["status"]), _ptr(lab) if lab is not None else None,
                                _ptr(scratch), scratch.numel(),
                                ctypes.c_void_p(streams[0].cuda_stream),
                                ctypes.c_void_p(streams[1].cuda_stream)), "tsa_segment_host")
    return out


# ------------------------------------------------------------------ 2-D
def make_problem2d(vol, bins, q, cluster=0):
    if vol.dim() != 3 or not vol.is_contiguous() or vol.dtype != torch.uint8:
        raise ValueError("2-D path: volume must be a contiguous uint8 [nz][ny][nx] tensor")
    nz, ny, nx = vol.shape
    return tsa2d_problem(vol.data_ptr(), nx, ny, nz, bins, float(q), cluster)


def tsa2d_cluster_size(vol, bins, q=0.8, cluster=0):
    return int(load().tsa2d_cluster_size(ctypes.byref(make_problem2d(vol, bins, q, cluster))))


def tsa2d_workspace(problem, device):
    n = int(load().tsa2d_workspace_size(ctypes.byref(problem)))
    if n == 0:
        _check(load().tsa2d_validate(ctypes.byref(problem)), "tsa2d_workspace_size")
    return torch.empty(n, dtype=torch.uint8, device=device)


def tsa2d_segment(vol, bins, q, labels=True, histogram=False, cluster=0, out=None, workspace=None,
                  stream=None):
    """2-D Tsallis path on the current stream.  Returns dict of
    device tensors: thresholds [nz,2] i32 (t, s), objective [nz] f64, status [nz]
    i32, labels [nz,ny,nx] u8 ([f > t]) or None, histogram [nz,bins,bins] or None."""
    _need_cuda(vol)
    p = make_problem2d(vol, bins, q, cluster)
    nz = vol.shape[0]
    dev = vol.device
    if out is None:
        out = {
            "thresholds": torch.empty((nz, 2), dtype=torch.int32, device=dev),
            "objective": torch.empty(nz, dtype=torch.float64, device=dev),
            "status": torch.empty(nz, dtype=torch.int32, device=dev),
            "labels": torch.empty(vol.shape, dtype=torch.uint8, device=dev) if labels else None,
            "histogram": (torch.empty((nz, bins, bins), dtype=torch.int32, device=dev)
                          if histogram else None),
        }
    o = tsa_outputs(out["thresholds"].data_ptr(),
                    out["labels"].data_ptr() if out.get("labels") is not None else None,
                    out["objective"].data_ptr() if out.get("objective") is not None else None,
                    out["histogram"].data_ptr() if out.get("histogram") is not None else None,
                    out["status"].data_ptr() if out.get("status") is not None else None)
    if workspace is None:
        workspace = tsa2d_workspace(p, dev)
    _check(load().tsa2d_segment(ctypes.byref(p), ctypes.byref(o), _ptr(workspace),
                                workspace.numel(), _stream(stream)), "tsa2d_segment")
    return out


def tsa2d_histogram(vol, bins, cluster=0, workspace=None, stream=None):
    _need_cuda(vol)
    p = make_problem2d(vol, bins, 1.0, cluster)
    nz = vol.shape[0]
    hist = torch.empty((nz, bins, bins), dtype=torch.int32, device=vol.device)
    status = torch.empty(nz, dtype=torch.int32, device=vol.device)
    if workspace is None:
        workspace = tsa2d_workspace(p, vol.device)
    _check(load().tsa2d_histogram(ctypes.byref(p), _ptr(hist), _ptr(status), _ptr(workspace),
                                  workspace.numel(), _stream(stream)), "tsa2d_histogram")
    return hist, status


def tsa2d_mean3x3(vol, stream=None):
    _need_cuda(vol)
    p = make_problem2d(vol, 256, 1.0)
    g = torch.empty(vol.shape, dtype=torch.uint8, device=vol.device)
    _check(load().tsa2d_mean3x3(ctypes.byref(p), _ptr(g), _stream(stream)), "tsa2d_mean3x3")
    return g


# --------------------------------------------------------------- HU input
def make_hu_problem(vol, k, q, background=-2000, objective="pseudo_additive",
                    enumeration="canonical"):
    if vol.dim() != 3 or not vol.is_contiguous() or vol.dtype != torch.int16:
        raise ValueError("HU path: volume must be a contiguous int16 [nz][ny][nx] tensor")
    nz, ny, nx = vol.shape
    return tsa_hu_problem(vol.data_ptr(), nx, ny, nz, int(background), k, float(q),
                          OBJECTIVES.get(objective, objective),
                          ENUMERATIONS.get(enumeration, enumeration))


def tsa_hu_workspace(problem, device):
    n = int(load().tsa_hu_workspace_size(ctypes.byref(problem)))
    if n == 0:
        raise TsaError(TSA_ERR_INVALID_ARG, "tsa_hu_workspace_size",
                       "HU problem: dims (nx*ny % 16), alignment, k, q or objective")
    return torch.empty(n, dtype=torch.uint8, device=device)


def tsa_hu_segment(vol, k, q, background=-2000, objective="pseudo_additive",
                   enumeration="canonical", labels=True, out=None, workspace=None, stream=None):
    """Pre-processing fused into the 1-D path (PAPER.md:514-516 then 558-597).
    Returns dict of device tensors: thresholds [nz,k] (8-bit levels), objective,
    histogram [nz,256] of the 8-bit image, status, labels, window [2] = (lo, hi) HU."""
    _need_cuda(vol)
    p = make_hu_problem(vol, k, q, background, objective, enumeration)
    nz = vol.shape[0]
    dev = vol.device
    if out is None:
        out = {
            "thresholds": torch.empty((nz, k), dtype=torch.int32, device=dev),
            "objective": torch.empty(nz, dtype=torch.float64, device=dev),
            "histogram": torch.empty((nz, 256), dtype=torch.int32, device=dev),
            "status": torch.empty(nz, dtype=torch.int32, device=dev),
            "labels": torch.empty(vol.shape, dtype=torch.uint8, device=dev) if labels else None,
            "window": torch.empty(2, dtype=torch.int32, device=dev),
        }
    o = tsa_outputs(out["thresholds"].data_ptr(),
                    out["labels"].data_ptr() if out.get("labels") is not None else None,
                    out["objective"].data_ptr() if out.get("objective") is not None else None,
                    out["histogram"].data_ptr() if out.get("histogram") is not None else None,
                    out["status"].data_ptr() if out.get("status") is not None else None)
    if workspace is None:
        workspace = tsa_hu_workspace(p, dev)
    win = out.get("window")
    _check(load().tsa_hu_segment(ctypes.byref(p), ctypes.byref(o), _ptr(win), _ptr(workspace),
                                 workspace.numel(), _stream(stream)), "tsa_hu_segment")
    return out


def tsa_hu_histogram(vol, k, q, background=-2000, objective="pseudo_additive",
                     enumeration="canonical", workspace=None, stream=None):
    """Phase 1 of tsa_hu_segment: HU histograms (kept in `workspace`) and the
    slab's window [2] = (lo, hi).  Returns (window, workspace)."""
    _need_cuda(vol)
    p = make_hu_problem(vol, k, q, background, objective, enumeration)
    if workspace is None:
        workspace = tsa_hu_workspace(p, vol.device)
    win = torch.empty(2, dtype=torch.int32, device=vol.device)
    _check(load().tsa_hu_histogram(ctypes.byref(p), _ptr(win), _ptr(workspace), workspace.numel(),
                                   _stream(stream)), "tsa_hu_histogram")
    return win, workspace


def tsa_hu_finish(vol, k, q, window, workspace, background=-2000, objective="pseudo_additive",
                  enumeration="canonical", labels=True, stream=None):
    """Phase 2: 8-bit histograms under the given (volume-wide) window, search,
    finalize, labels.  Returns the dict of tsa_hu_segment (without "window")."""
    _need_cuda(vol, window, workspace)
    p = make_hu_problem(vol, k, q, background, objective, enumeration)
    nz = vol.shape[0]
    dev = vol.device
    out = {
        "thresholds": torch.empty((nz, k), dtype=torch.int32, device=dev),
        "objective": torch.empty(nz, dtype=torch.float64, device=dev),
        "histogram": torch.empty((nz, 256), dtype=torch.int32, device=dev),
        "status": torch.empty(nz, dtype=torch.int32, device=dev),
        "labels": torch.empty(vol.shape, dtype=torch.uint8, device=dev) if labels else None,
    }
    o = tsa_outputs(out["thresholds"].data_ptr(),
                    out["labels"].data_ptr() if out["labels"] is not None else None,
                    out["objective"].data_ptr(), out["histogram"].data_ptr(), out["status"].data_ptr())
    _check(load().tsa_hu_finish(ctypes.byref(p), _ptr(window), ctypes.byref(o), _ptr(workspace),
                                workspace.numel(), _stream(stream)), "tsa_hu_finish")
    return out


def tsa_hu_preprocess(vol, background=-2000, workspace=None, stream=None):
    """The 8-bit image alone: (gray [nz,ny,nx] u8, window [2] = (lo, hi))."""
    _need_cuda(vol)
    p = make_hu_problem(vol, 1, 1.0, background)
    gray = torch.empty(vol.shape, dtype=torch.uint8, device=vol.device)
    win = torch.empty(2, dtype=torch.int32, device=vol.device)
    if workspace is None:
        workspace = tsa_hu_workspace(p, vol.device)
    _check(load().tsa_hu_preprocess(ctypes.byref(p), _ptr(gray), _ptr(win), _ptr(workspace),
                                    workspace.numel(), _stream(stream)), "tsa_hu_preprocess")
    return gray, win


# ------------------------------------------------------------- morphology
MORPH_OPS = {"erode": 0, "dilate": 1, "open": 2, "tophat": 3}


def tsa_morph(vol, op="tophat", radius=10, out=None, workspace=None, stream=None):
    """Disk(radius) grayscale morphology per slice:
    'erode', 'dilate', 'open' or 'tophat' (max(vol - open(vol), 0))."""
    _need_cuda(vol)
    if vol.dim() != 3 or not vol.is_contiguous() or vol.dtype != torch.uint8:
        raise ValueError("morphology: volume must be a contiguous uint8 [nz][ny][nx] tensor")
    nz, ny, nx = vol.shape
    code = MORPH_OPS.get(op, op)
    if out is None:
        out = torch.empty_like(vol)
    n = int(load().tsa_morph_workspace_size(nx, ny, nz, code))
    if workspace is None and n:
        workspace = torch.empty(n, dtype=torch.uint8, device=vol.device)
    _check(load().tsa_morph(_ptr(vol), _ptr(out), nx, ny, nz, int(radius), code, _ptr(workspace),
                            workspace.numel() if workspace is not None else 0, _stream(stream)),
           "tsa_morph")
    return out


def tsa_class_consts(n, q, stream=None):
    """The class-size constants of the search kernels for class sizes `n`
    (u32 values in an int32/int64 CUDA tensor): n^-q (q != 1) or (ln n, 1/n)
    (q == 1).  Returns a (or (a, b) at q == 1) as f64 CUDA tensors."""
    _need_cuda(n)
    lib = load()
    n32 = n.to(torch.int32).contiguous()
    a = torch.empty(n32.shape, dtype=torch.float64, device=n.device)
    b = torch.empty(n32.shape, dtype=torch.float64, device=n.device) if q == 1.0 else None
    ws = torch.empty(int(lib.tsa_class_consts_workspace_size()), dtype=torch.uint8, device=n.device)
    _check(lib.tsa_class_consts(_ptr(n32), n32.numel(), float(q), _ptr(a), _ptr(b), _ptr(ws), ws.numel(),
                                _stream(stream)), "tsa_class_consts")
    return (a, b) if b is not None else a


def unpack_key(key, k):
    """Packed u64 key (as python int) -> tuple of k thresholds."""
    key &= 0xFFFFFFFFFFFFFFFF
    return tuple((key >> (12 * (k - 1 - j))) & 0xFFF for j in range(k))


# ------------------------------------------------------------------ q sweep
def tsa_segment_sweep(vol, bins, k, qs, objective="pseudo_additive", enumeration="canonical",
                      units=0, labels=True, outs=None, workspace=None, stream=None):
    """One histogram, then search / finalize / labels for every q in `qs`
    (tsa_segment_sweep).  Returns a list of per-q output dicts (as tsa_segment)."""
    _need_cuda(vol)
    lib = load()
    qs = [float(x) for x in qs]
    p = make_problem(vol, bins, k, qs[0], objective, enumeration, units)
    nz, dev = vol.shape[0], vol.device
    if outs is None:
        hist = torch.empty((nz, bins), dtype=torch.int32, device=dev)
        outs = [{"thresholds": torch.empty((nz, k), dtype=torch.int32, device=dev),
                 "objective": torch.empty(nz, dtype=torch.float64, device=dev),
                 "histogram": hist if i == 0 else None,
                 "status": torch.empty(nz, dtype=torch.int32, device=dev),
                 "labels": torch.empty(vol.shape, dtype=torch.uint8, device=dev) if labels else None}
                for i in range(len(qs))]
    qa = (ctypes.c_double * len(qs))(*qs)
    oa = (tsa_outputs * len(qs))()
    for i, o in enumerate(outs):
        oa[i] = tsa_outputs(o["thresholds"].data_ptr(),
                            o["labels"].data_ptr() if o.get("labels") is not None else None,
                            o["objective"].data_ptr() if o.get("objective") is not None else None,
                            o["histogram"].data_ptr() if o.get("histogram") is not None else None,
                            o["status"].data_ptr() if o.get("status") is not None else None)
    if workspace is None:
        n = int(lib.tsa_sweep_workspace_size(ctypes.byref(p), qa, len(qs)))
        if n == 0:
            _check(TSA_ERR_INVALID_ARG, "tsa_sweep_workspace_size")
        workspace = torch.empty(n, dtype=torch.uint8, device=dev)
    _check(lib.tsa_segment_sweep(ctypes.byref(p), qa, len(qs), oa, _ptr(workspace), workspace.numel(),
                                 _stream(stream)), "tsa_segment_sweep")
    return outs


def sweep_workspace(vol, bins, k, qs, objective="pseudo_additive", enumeration="canonical", units=0):
    p = make_problem(vol, bins, k, float(qs[0]), objective, enumeration, units)
    qa = (ctypes.c_double * len(qs))(*[float(x) for x in qs])
    n = int(load().tsa_sweep_workspace_size(ctypes.byref(p), qa, len(qs)))
    return torch.empty(max(n, 1), dtype=torch.uint8, device=vol.device)


# ---------------------------------------------------------------- multi-GPU
def tsa_slab_range(nz_total, nranks, rank):
    z0, z1 = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(load().tsa_slab_range(nz_total, nranks, rank, ctypes.byref(z0), ctypes.byref(z1)),
           "tsa_slab_range")
    return z0.value, z1.value


def tsa_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(COMM_ID_BYTES)
    _check(load().tsa_comm_unique_id(buf), "tsa_comm_unique_id")
    return buf.raw


class TsaComm:
    """Owner of a libtsa communicator (tsa_comm_init / tsa_comm_init_custom).
    ``TsaComm.nccl(nranks, rank, uid)`` (uid: tsa_comm_unique_id() of rank 0,
    distributed by the caller) or ``TsaComm.custom(nranks, rank, fn)`` with
    fn(send_ptr, recv_ptr, nbytes, stream_handle) -> None (raise on error)."""

    def __init__(self, handle, nranks, rank, keep=None):
        self.handle, self.nranks, self.rank, self._keep = handle, nranks, rank, keep

    @classmethod
    def nccl(cls, nranks, rank, uid: bytes):
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(uid, COMM_ID_BYTES)
        _check(load().tsa_comm_init(ctypes.byref(h), nranks, rank, buf), "tsa_comm_init")
        return cls(h, nranks, rank)

    @classmethod
    def custom(cls, nranks, rank, fn):
        def tramp(user, send, recv, nbytes, stream):
            try:
                fn(send, recv, nbytes, stream)
                return 0
            except Exception:  # reported as TSA_ERR_NCCL by the library
                import traceback

                traceback.print_exc()
                return 1

        cb = ALLGATHER_FN(tramp)
        h = ctypes.c_void_p()
        _check(load().tsa_comm_init_custom(ctypes.byref(h), nranks, rank, cb, None), "tsa_comm_init_custom")
        return cls(h, nranks, rank, keep=cb)

    @property
    def kind(self):
        return int(load().tsa_comm_kind(self.handle))

    def close(self):
        if self.handle:
            _check(load().tsa_comm_destroy(self.handle), "tsa_comm_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tsa_segment_sharded(slab, nz_total, bins, k, q, comm, mode="tuples", objective="pseudo_additive",
                        enumeration="canonical", units=0, labels=True, workspace=None, stream=None,
                        nx=None, ny=None, dtype=torch.uint8):
    """tsa_segment_sharded: `slab` is this rank's slices (tsa_slab_range of
    nz_total) on this rank's GPU (may have 0 slices in tuples mode; pass
    nx/ny/dtype then).  tuples mode: thresholds/objective/status/histogram for
    all nz_total slices (identical on every rank) + the own slab's labels;
    slices mode: everything for the own slab (no exchange)."""
    _need_cuda(slab)
    lib = load()
    m = SHARD_MODES.get(mode, mode)
    dev = slab.device
    n_own = slab.shape[0]
    ny = slab.shape[1] if ny is None else ny
    nx = slab.shape[2] if nx is None else nx
    p = tsa_problem(slab.data_ptr() if n_own > 0 else None,
                    _dtype_code(slab) if n_own > 0 else (TSA_U8 if dtype == torch.uint8 else TSA_U16),
                    nx, ny, n_own, bins, k, float(q), OBJECTIVES.get(objective, objective),
                    ENUMERATIONS.get(enumeration, enumeration), units, 0, 0, 0)
    nres = n_own if m == TSA_SHARD_SLICES else nz_total
    out = {"thresholds": torch.empty((nres, k), dtype=torch.int32, device=dev),
           "objective": torch.empty(nres, dtype=torch.float64, device=dev),
           "histogram": torch.empty((nres, bins), dtype=torch.int32, device=dev),
           "status": torch.empty(nres, dtype=torch.int32, device=dev),
           "labels": torch.empty((n_own, ny, nx), dtype=torch.uint8, device=dev) if labels else None}
    o = tsa_outputs(out["thresholds"].data_ptr(),
                    out["labels"].data_ptr() if labels and n_own > 0 else None,
                    out["objective"].data_ptr(), out["histogram"].data_ptr(), out["status"].data_ptr())
    if workspace is None:
        n = int(lib.tsa_sharded_workspace_size(ctypes.byref(p), nz_total, m, comm.handle))
        workspace = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    _check(lib.tsa_segment_sharded(ctypes.byref(p), nz_total, ctypes.byref(o), m, comm.handle,
                                   _ptr(workspace), workspace.numel(), _stream(stream)),
           "tsa_segment_sharded")
    out["units"] = int(lib.tsa_sharded_units(ctypes.byref(p), nz_total, comm.nranks))
    return out
