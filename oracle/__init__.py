"""CPU oracle for the abin hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct implementation of what arXiv 1905.13038's
method computes, written from the paper's definitions
(see abin_oracle.c for the per-function citations).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product package paper_1905_13038_b200 never
imports it, and the two share no code.

Parity unpinned (no paper value fixes them, DESIGN.md lists the readings):
the exact fp64 bits of t beyond the literal Table-1 order, and the quantile
rank convention rho = max(1, ceil(q n)).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "abin_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
# -ffp-contract=off / -fno-fast-math: IEEE double evaluated literally, no FMA
# contraction (reading R5).
CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]

SAUVOLA, NIBLACK, WOLF = 0, 1, 2
_METHODS = {"sauvola": SAUVOLA, "niblack": NIBLACK, "wolf": WOLF}
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.orc_offsets.argtypes = [_I32, _I32, _P]
        lib.orc_count.argtypes = [_I64, _I64, _I32, _I32, _I64, _I64]
        lib.orc_count.restype = _I64
        lib.orc_threshold.argtypes = [_I32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _D, _D, _D]
        lib.orc_threshold.restype = _D
        lib.orc_global_min.argtypes = [_P, _I64, _I64, _I64]
        lib.orc_global_min.restype = _I32
        lib.orc_binarize.argtypes = [_I32, _P, _I64, _I64, _I64, _I32, _I32, _D, _D, _I32, _P, _P, _P, _P, _P, _P]
        lib.orc_binarize_points.argtypes = [_I32, _P, _I64, _I64, _I64, _I32, _I32, _D, _D, _I32, _I64, _P, _P,
                                            _P, _P, _P, _P, _P]
        lib.orc_max_s.argtypes = [_P, _I64, _I64, _I64, _I32, _I32]
        lib.orc_max_s.restype = _D
        lib.orc_adaptive_R.argtypes = [_D]
        lib.orc_adaptive_R.restype = _D
        lib.orc_alg1_stats.argtypes = [_P, _I64, _I64, _I64, _I32, _I32, _P, _P]
        lib.orc_integral_stats.argtypes = [_P, _I64, _I64, _I64, _I32, _I32, _P, _P]
        lib.orc_quantile.argtypes = [_P, _I64, _I64, _I64, _I32, _I32, _D, _P, _P]
        lib.orc_quantile_points.argtypes = [_P, _I64, _I64, _I64, _I32, _I32, _D, _I64, _P, _P, _P, _P]
        lib.orc_bernsen.argtypes = [_P, _I64, _I64, _I64, _I32, _I32, _I32, _P, _P, _P]
        lib.orc_bernsen_points.argtypes = [_P, _I64, _I64, _I64, _I32, _I32, _I32, _I64, _P, _P, _P]
        lib.orc_threshold_rule.argtypes = [_I32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _P, _D, _D, _D,
                                           _D]
        lib.orc_threshold_rule.restype = _D
        lib.orc_global_mean_std.argtypes = [_P, _I64, _I64, _I64, _P, _P]
        lib.orc_binarize_rule.argtypes = [_I32, _P, _I64, _I64, _I64, _I32, _I32, _P, _I64, _P, _P, _P, _P]
        lib.orc_otsu.argtypes = [_P, _I64, _I64, _I64]
        lib.orc_otsu.restype = _I32
        lib.orc_num_threads.restype = ctypes.c_int
        lib.orc_set_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _img(I):
    I = np.asarray(I)
    assert I.dtype == np.uint8 and I.ndim == 2 and I.strides[1] == 1
    return I


def _ptr(a):
    return None if a is None else a.ctypes.data


def num_threads() -> int:
    return _load().orc_num_threads()


def set_threads(n: int) -> None:
    _load().orc_set_threads(n)


def offsets(h: int, w: int):
    """(l, r, o, u) of Alg. 1 l.1-4."""
    out = np.zeros(4, dtype=np.int64)
    _load().orc_offsets(h, w, out.ctypes.data)
    return tuple(int(x) for x in out)


def count(H, W, h, w, i, j) -> int:
    """n of Alg. 1 l.118."""
    return int(_load().orc_count(H, W, h, w, i, j))


def threshold(method: str, c: int, d: int, n: int, k: float, R: float = 128.0, L: float = 0.0) -> float:
    """Canonical fp64 threshold from exact (c, d, n) -- Table 1, left to right."""
    return float(_load().orc_threshold(_METHODS[method], c, d, n, k, R, L))


def max_s(I, h: int, w: int) -> float:
    """Wolf's adaptive R source: max over the page of the canonical fp64 s."""
    I = _img(I)
    return _load().orc_max_s(I.ctypes.data, I.shape[0], I.shape[1], I.strides[0], h, w)


def adaptive_R(I, h: int, w: int) -> float:
    """R = max s, or +inf when every window is constant (R21)."""
    return _load().orc_adaptive_R(max_s(I, h, w))


def global_min(I) -> int:
    I = _img(I)
    return int(_load().orc_global_min(I.ctypes.data, I.shape[0], I.shape[1], I.strides[0]))


def binarize(method: str, I, h: int, w: int, k: float, R: float = 128.0, L: int = -1, stats: bool = False):
    """Direct Theta(HWhw) binarization.  Returns mask (uint8 0 = foreground) or,
    with stats=True, a dict with mask, c, d, n, t and near_tie."""
    I = _img(I)
    H, W = I.shape
    mask = np.empty((H, W), np.uint8)
    c = d = n = t = None
    if stats:
        c = np.empty((H, W), np.uint64)
        d = np.empty((H, W), np.uint64)
        n = np.empty((H, W), np.uint64)
        t = np.empty((H, W), np.float64)
    ties = np.zeros(1, np.uint64)
    _load().orc_binarize(_METHODS[method], I.ctypes.data, H, W, I.strides[0], h, w, k, R, L, mask.ctypes.data,
                         _ptr(c), _ptr(d), _ptr(n), _ptr(t), ties.ctypes.data)
    if not stats:
        return mask
    return {"mask": mask, "c": c, "d": d, "n": n, "t": t, "near_tie": int(ties[0])}


def binarize_points(method: str, I, h: int, w: int, k: float, R: float, L: int, rows, cols):
    """The definition evaluated at sampled pixels only (full-size parity)."""
    I = _img(I)
    H, W = I.shape
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    m = rows.size
    if method == "wolf" and L < 0:
        L = global_min(I)
    out = {"mask": np.empty(m, np.uint8), "c": np.empty(m, np.uint64), "d": np.empty(m, np.uint64),
           "n": np.empty(m, np.uint64), "t": np.empty(m, np.float64)}
    _load().orc_binarize_points(_METHODS[method], I.ctypes.data, H, W, I.strides[0], h, w, k, R, L, m,
                                rows.ctypes.data, cols.ctypes.data, out["mask"].ctypes.data,
                                out["c"].ctypes.data, out["d"].ctypes.data, out["n"].ctypes.data,
                                out["t"].ctypes.data)
    return out


def alg1_stats(I, h: int, w: int):
    """(c, d) per pixel by a literal transcription of Algorithm 1's recursion."""
    I = _img(I)
    H, W = I.shape
    c = np.empty((H, W), np.uint64)
    d = np.empty((H, W), np.uint64)
    if _load().orc_alg1_stats(I.ctypes.data, H, W, I.strides[0], h, w, c.ctypes.data, d.ctypes.data) != 0:
        raise MemoryError
    return c, d


def integral_stats(I, h: int, w: int):
    """(c, d) per pixel through Sec. 2 integral images."""
    I = _img(I)
    H, W = I.shape
    c = np.empty((H, W), np.uint64)
    d = np.empty((H, W), np.uint64)
    if _load().orc_integral_stats(I.ctypes.data, H, W, I.strides[0], h, w, c.ctypes.data, d.ctypes.data) != 0:
        raise MemoryError
    return c, d


def quantile(I, h: int, w: int, q: float):
    """Direct sort-based local quantile.  Returns (mask, Q)."""
    I = _img(I)
    H, W = I.shape
    mask = np.empty((H, W), np.uint8)
    Q = np.empty((H, W), np.uint8)
    if _load().orc_quantile(I.ctypes.data, H, W, I.strides[0], h, w, q, mask.ctypes.data, Q.ctypes.data) != 0:
        raise MemoryError
    return mask, Q


def quantile_points(I, h: int, w: int, q: float, rows, cols):
    I = _img(I)
    H, W = I.shape
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    m = rows.size
    mask = np.empty(m, np.uint8)
    Q = np.empty(m, np.uint8)
    if _load().orc_quantile_points(I.ctypes.data, H, W, I.strides[0], h, w, q, m, rows.ctypes.data,
                                   cols.ctypes.data, mask.ctypes.data, Q.ctypes.data) != 0:
        raise MemoryError
    return mask, Q


def bernsen(I, h: int, w: int, contrast: int = -1):
    """Bernsen midrange rule: mask 0 iff 2 I <= min + max of the
    in-bounds window; contrast >= 0: background where max - min < contrast.
    Returns (mask, min, max)."""
    I = _img(I)
    H, W = I.shape
    mask = np.empty((H, W), np.uint8)
    lo = np.empty((H, W), np.uint8)
    hi = np.empty((H, W), np.uint8)
    _load().orc_bernsen(I.ctypes.data, H, W, I.strides[0], h, w, contrast, mask.ctypes.data, lo.ctypes.data,
                        hi.ctypes.data)
    return mask, lo, hi


def bernsen_points(I, h: int, w: int, contrast: int, rows, cols):
    I = _img(I)
    H, W = I.shape
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    mask = np.empty(rows.size, np.uint8)
    _load().orc_bernsen_points(I.ctypes.data, H, W, I.strides[0], h, w, contrast, rows.size, rows.ctypes.data,
                               cols.ctypes.data, mask.ctypes.data)
    return mask


RULES = {"feng": 5, "rais": 6, "khurshid": 7, "phansalkar": 8}


def threshold_rule(rule: str, c: int, d: int, n: int, params=(), L: float = 0.0, M: float = 0.0, S: float = 0.0,
                   hw: float = 1.0) -> float:
    """Table 1 rows Feng / Rais / Khurshid / Phansalkar, canonical fp64."""
    prm = np.ascontiguousarray(list(params) + [0.0] * (8 - len(params)), dtype=np.float64)
    return _load().orc_threshold_rule(RULES[rule], c, d, n, prm.ctypes.data, L, M, S, hw)


def global_mean_std(I):
    I = _img(I)
    M, S = ctypes.c_double(), ctypes.c_double()
    _load().orc_global_mean_std(I.ctypes.data, I.shape[0], I.shape[1], I.strides[0], ctypes.byref(M), ctypes.byref(S))
    return M.value, S.value


def binarize_rule(rule: str, I, h: int, w: int, params=(), rows=None, cols=None, with_t: bool = False):
    """Mask (and t) of a Table 1 rule on the whole page, or at sampled pixels."""
    I = _img(I)
    H, W = I.shape
    prm = np.ascontiguousarray(list(params) + [0.0] * (8 - len(params)), dtype=np.float64)
    if rows is None:
        m, rp, cp = H * W, None, None
        shape = (H, W)
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        m, rp, cp = rows.size, rows.ctypes.data, cols.ctypes.data
        shape = (rows.size,)
    mask = np.empty(shape, np.uint8)
    t = np.empty(shape, np.float64)
    _load().orc_binarize_rule(RULES[rule], I.ctypes.data, H, W, I.strides[0], h, w, prm.ctypes.data, m, rp, cp,
                              mask.ctypes.data, t.ctypes.data)
    return (mask, t) if with_t else mask


def otsu(I):
    """Otsu's global threshold t and the mask (0 iff I <= t)."""
    I = _img(I)
    t = int(_load().orc_otsu(I.ctypes.data, I.shape[0], I.shape[1], I.strides[0]))
    return t, (I > t).astype(np.uint8)


def pack_bits(mask: np.ndarray) -> np.ndarray:
    """MSB-first bit packing of a 0/1 mask, rows padded to whole bytes."""
    return np.packbits(mask.astype(np.uint8), axis=-1, bitorder="big")
