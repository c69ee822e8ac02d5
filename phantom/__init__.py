"""Seeded synthetic CT phantom (the input generator shared by the CUDA path's
tests/bench and the oracle).  Holds none of the method's arithmetic.

``make_volume(cfg)`` returns a numpy ``[nz][ny][nx]`` u8/u16 volume; the C
generator lives in ``phantom.c`` (recipe in its header and DESIGN.md).
``CONFIGS`` are the five workloads of BASELINE.json:configs.
"""
from __future__ import annotations

import ctypes
import dataclasses
import hashlib
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libphantom.so")
_SRC = os.path.join(_HERE, "phantom.c")

SEED_BASE = 2012106840


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _SO, _SRC, "-lm"]
        )
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.phantom_generate.restype = ctypes.c_int
        lib.phantom_generate.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int,
        ]
        _lib = lib
    return _lib


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    nx: int
    ny: int
    nz: int
    dtype: str  # "u8" | "u16" | "i16" (raw HU)
    bins: int
    k: int
    qs: tuple
    seed: int
    z_first: int = 0
    z_total: int = 0  # 0 -> nz
    note: str = ""

    @property
    def np_dtype(self):
        return {"u8": np.uint8, "u16": np.uint16, "i16": np.int16}[self.dtype]

    @property
    def depth(self):
        return self.z_total or self.nz


CONFIGS = {
    # single 256x256 8-bit slice at carina level (40 % of a 300-slice phantom)
    "c1": Config("c1", 256, 256, 1, "u8", 256, 1, (0.8,), SEED_BASE + 1, z_first=120,
                 z_total=300, note="single 256x256 8-bit slice, 256 bins, k=1, q=0.8"),
    "c2": Config("c2", 512, 512, 300, "u8", 256, 2, (0.8,), SEED_BASE + 2,
                 note="512x512x300 phantom, 256 bins, k=2"),
    "c3": Config("c3", 512, 512, 600, "u8", 256, 3,
                 tuple(round(0.5 + 0.1 * i, 1) for i in range(11)), SEED_BASE + 3,
                 note="512x512x600 phantom, 256 bins, k=3, q sweep 0.5..1.5"),
    "c4": Config("c4", 512, 512, 300, "u8", 256, 4, (0.8,), SEED_BASE + 4,
                 note="512x512x300 phantom, 256 bins, k=4, tuple-sharded"),
    "c5": Config("c5", 1024, 1024, 1000, "u16", 4096, 2, (0.8,), SEED_BASE + 5,
                 note="1024x1024x1000 12-bit phantom, 4096 bins, k=2"),
    # the paper's 2-D formulation on the c2 volume (same
    # seed and bytes); k = 1 stands for the single (t, s) pair
    # raw int16 HU of the c2 phantom (background -2000),
    # pre-processed to 8 bits inside the histogram / label passes
    "f2": Config("f2", 512, 512, 300, "i16", 256, 2, (0.8,), SEED_BASE + 2,
                 note="HU int16 512x512x300 phantom (c2 geometry), pre-processing fused: "
                      "background -2000 -> 0, volume-wide linear rescale to 0..255, 256 bins, k=2"),
    # disk(10) opening + white top-hat (the chest mask,
    # PAPER.md:528-550) of the c2 volume; k = 10 stands for the disk radius
    "f3": Config("f3", 512, 512, 300, "u8", 256, 10, (0.8,), SEED_BASE + 2,
                 note="disk(10) opening + white top-hat of the 512x512x300 c2 phantom"),
    "f1": Config("f1", 512, 512, 300, "u8", 256, 1, (0.8,), SEED_BASE + 2,
                 note="2-D Tsallis (PAPER.md:564-597) on the 512x512x300 c2 phantom, 256 levels, "
                      "(t,s) search, q=0.8"),
}


def generate(nx, ny, nz, dtype="u8", seed=SEED_BASE, z_first=0, z_total=0, threads=None, out=None):
    lib = _load()
    npdt = {"u8": np.uint8, "u16": np.uint16, "i16": np.int16}[dtype]
    if out is None:
        out = np.empty((nz, ny, nx), dtype=npdt)
    assert out.flags.c_contiguous and out.dtype == npdt and out.shape == (nz, ny, nx)
    threads = threads or os.cpu_count() or 1
    rc = lib.phantom_generate(out.ctypes.data, {"u8": 1, "u16": 2, "i16": 3}[dtype], nx, ny, nz,
                              z_first, z_total or nz, seed, threads)
    if rc != 0:
        raise ValueError("phantom_generate failed")
    return out


def make_volume(cfg: Config, nz: int | None = None, z_first: int | None = None, out=None):
    """The config's volume (optionally a sub-slab [z_first, z_first+nz))."""
    zf = cfg.z_first if z_first is None else cfg.z_first + z_first
    n = cfg.nz if nz is None else nz
    return generate(cfg.nx, cfg.ny, n, cfg.dtype, cfg.seed, zf, cfg.depth, out=out)


def sha256(vol: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(vol).tobytes()).hexdigest()
