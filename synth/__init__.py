"""Seeded synthetic document pages -- the shared input generator.

This module draws the BASELINE.json workloads' pixels (see synth.c for the
recipe) and nothing else: it holds none of the method's arithmetic, so both
the oracle side (tests) and the product side (bench.py) may use it.

Seeds follow DESIGN.md: page p of config `cfg` uses 1905130380 + 1000*cfg + p.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")
_lib = None

SEED_BASE = 1905130380


def config_seed(cfg: int, page: int = 0) -> int:
    return SEED_BASE + 1000 * cfg + page


def build(force: bool = False) -> str:
    """Compile synth.c -> libsynth.so (gcc, OpenMP)."""
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.synth_page.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                   ctypes.c_void_p, ctypes.c_int64]
        lib.synth_page.restype = ctypes.c_int
        lib.synth_pages.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64]
        lib.synth_pages.restype = ctypes.c_int
        lib.synth_hash.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        lib.synth_hash.restype = ctypes.c_uint64
        _lib = lib
    return _lib


def page(H: int, W: int, seed: int, stain: bool = False, out: np.ndarray = None) -> np.ndarray:
    """One H x W uint8 page (C-contiguous, or written into `out`)."""
    lib = _load()
    if out is None:
        out = np.empty((H, W), dtype=np.uint8)
    assert out.dtype == np.uint8 and out.shape[-2:] == (H, W) and out.strides[-1] == 1
    rc = lib.synth_page(seed, H, W, 1 if stain else 0, out.ctypes.data, out.strides[-2])
    if rc != 0:
        raise MemoryError("synth_page failed")
    return out


def pages(P: int, H: int, W: int, seed0: int, stain: bool = False, out: np.ndarray = None) -> np.ndarray:
    """P pages as a (P, H, W) uint8 array; page p uses seed0 + p."""
    lib = _load()
    if out is None:
        out = np.empty((P, H, W), dtype=np.uint8)
    assert out.dtype == np.uint8 and out.shape == (P, H, W) and out.strides[-1] == 1
    rc = lib.synth_pages(seed0, P, H, W, 1 if stain else 0, out.ctypes.data, out.strides[1], out.strides[0])
    if rc != 0:
        raise MemoryError("synth_pages failed")
    return out


def page_hash(img: np.ndarray) -> int:
    """FNV-1a 64 over the page's pixels in row-major order."""
    lib = _load()
    assert img.dtype == np.uint8 and img.ndim == 2 and img.strides[-1] == 1
    return int(lib.synth_hash(img.ctypes.data, img.shape[0], img.shape[1], img.strides[0]))


# ---- adversarial / degenerate inputs used by the parity tests -------------

def uniform_random(H: int, W: int, seed: int, lo: int = 0, hi: int = 255) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(lo, hi + 1, size=(H, W), dtype=np.uint8)


def low_contrast(H: int, W: int, seed: int, centre: int = 128, spread: int = 2) -> np.ndarray:
    """centre +- spread: puts Niblack thresholds within ~1e-13 of pixel values."""
    return uniform_random(H, W, seed, centre - spread, centre + spread)


def constant(H: int, W: int, g: int) -> np.ndarray:
    return np.full((H, W), g, dtype=np.uint8)
