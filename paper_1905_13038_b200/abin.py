"""Thin Python binding of libabin.so (include/abin.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  Tensors are torch CUDA uint8 tensors (device
memory, streams and process groups are all PyTorch provides here).  There is
no CPU fallback: if the shared library is missing, importing this module
raises.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ABIN_LIB", os.path.join(_HERE, "libabin.so"))  # ABIN_LIB: dev A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = ctypes.CDLL(LIB_PATH)

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U32 = ctypes.c_uint32
_D = ctypes.c_double

SAUVOLA, NIBLACK, WOLF, QUANTILE, BERNSEN = 0, 1, 2, 3, 4
METHODS = {"sauvola": SAUVOLA, "niblack": NIBLACK, "wolf": WOLF, "quantile": QUANTILE, "bernsen": BERNSEN}
MASK_U8, MASK_BITS = 0, 1
FORCE_U64_SQ, FORCE_FP64, HOST_IO, COUNT_STAGES = 1, 2, 4, 8
V4_INTERNAL = 1 << 27  # internal test hook: the v4 warp-CTA kernel instead of v5 (A/B parity)
Q2_INTERNAL = 1 << 26  # internal test hook: the round-1 quantile kernels instead of v5 (A/B parity)
V3_INTERNAL = 1 << 29  # internal test hook: the 4-warp-CTA kernel instead of the warp-CTA kernel
NO_TMA_INTERNAL = 1 << 30  # internal test hook: the generic row loader (no TMA, no re-pitched copy)
OK, EINVAL, EALIAS, ERANGE, ECUDA, ENOMEM = 0, 1, 2, 3, 4, 5

_lib.abin_sauvola.argtypes = [_P, _I64, _I64, _I64, _P, _I64, _I32, _I32, _I32, _D, _D, _U32, _P, _P]
_lib.abin_niblack.argtypes = [_P, _I64, _I64, _I64, _P, _I64, _I32, _I32, _I32, _D, _U32, _P, _P]
_lib.abin_wolf.argtypes = [_P, _I64, _I64, _I64, _P, _I64, _I32, _I32, _I32, _D, _D, _I32, _U32, _P, _P]
_lib.abin_quantile.argtypes = [_P, _I64, _I64, _I64, _P, _I64, _I32, _I32, _I32, _D, _U32, _P]
_lib.abin_bernsen.argtypes = [_P, _I64, _I64, _I64, _P, _I64, _I32, _I32, _I32, _I32, _U32, _P]
_lib.abin_binarize_rule.argtypes = [_I32, _P, _I64, _I64, _I64, _P, _I64, _I32, _I32, _I32, _P, _I32, _U32, _P, _P]
RULES = {"feng": 5, "rais": 6, "khurshid": 7, "phansalkar": 8}
_lib.abin_otsu.argtypes = [_P, _I64, _I64, _I64, _P, _I64, _I32, _P, _U32, _P]
_lib.abin_binarize_batched.argtypes = [_I32, _P, _I64, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _I32, _I32, _D,
                                       _D, _I32, _U32, _P, _P]
_lib.abin_binarize_band.argtypes = [_I32, _P, _I64, _I64, _I64, _I64, _I64, _I32, _I32, _P, _I64, _I32, _I32, _I32,
                                    _D, _D, _I32, _U32, _P, _P]
_lib.abin_global_min.argtypes = [_P, _I64, _I64, _I64, _I64, _I64, _P, _P]
_lib.abin_stats.argtypes = [_I32, _P, _I64, _I64, _I64, _I32, _I32, _D, _D, _I32, _P, _P, _P, _P, _P, _P]
_lib.abin_max_s.argtypes = [_P, _I64, _I64, _I64, _I64, _I64, _I32, _I32, _I32, _I32, _P, _P]
_lib.abin_wolf_adaptive.argtypes = [_P, _I64, _I64, _I64, _P, _I64, _I32, _I32, _I32, _D, _I32, _U32, _P, _P, _P]
_lib.abin_probe_filter.argtypes = [_I32, _D, _D, _D, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P]
_lib.abin_strerror.argtypes = [ctypes.c_int]
_lib.abin_strerror.restype = ctypes.c_char_p
_lib.abin_version.restype = ctypes.c_char_p
_lib.abin_last_cuda_error.restype = ctypes.c_char_p


class AbinLimits(ctypes.Structure):
    _fields_ = [("max_window_w", _I64), ("max_window_h", _I64), ("max_window_hw", _I64), ("max_dim", _I64),
                ("quantile_max_window_w", _I64), ("quantile_max_window_hw", _I64),
                ("bernsen_max_window_w", _I64)]


_lib.abin_limits.argtypes = [ctypes.POINTER(AbinLimits)]

EXPORTED = ["abin_sauvola", "abin_niblack", "abin_wolf", "abin_quantile", "abin_bernsen", "abin_binarize_rule", "abin_otsu",
            "abin_binarize_batched",
            "abin_binarize_band", "abin_global_min", "abin_stats", "abin_limits", "abin_strerror", "abin_version",
            "abin_last_cuda_error", "abin_probe_filter", "abin_max_s", "abin_wolf_adaptive"]


class AbinError(RuntimeError):
    def __init__(self, status: int):
        msg = _lib.abin_strerror(status).decode()
        if status == ECUDA:
            msg += ": " + _lib.abin_last_cuda_error().decode()
        super().__init__(f"abin status {status}: {msg}")
        self.status = status


def _check(rc: int) -> None:
    if rc != OK:
        raise AbinError(rc)


def version() -> str:
    return _lib.abin_version().decode()


def limits() -> AbinLimits:
    out = AbinLimits()
    _lib.abin_limits(ctypes.byref(out))
    return out


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(stream, device=None):
    """The caller's stream as a raw cudaStream_t (int).  With no stream given:
    the current stream of `device` (the call's tensor device) -- read with
    torch's raw-stream accessor, a tenth of torch.cuda.current_stream()'s
    host cost (a few microseconds per call on the small pages)."""
    if stream is not None:
        return stream.cuda_stream
    if _raw_stream is not None:
        return _raw_stream(torch.cuda.current_device() if device is None else device)
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _img2d(x: torch.Tensor):
    if x.dtype != torch.uint8 or x.dim() != 2 or not x.is_cuda or x.stride(1) != 1:
        raise ValueError("expected a 2-D CUDA uint8 tensor with unit column stride")
    return x.shape[0], x.shape[1], x.stride(0)


def _alloc_mask(H, W, packed, device, pitch=None):
    cols = (W + 7) // 8 if packed else W
    if pitch is None:
        return torch.empty((H, cols), dtype=torch.uint8, device=device)
    buf = torch.empty((H, pitch), dtype=torch.uint8, device=device)
    return buf[:, :cols]


def sauvola(img: torch.Tensor, h: int, w: int, k: float = 0.5, R: float = 128.0, packed: bool = False, out=None,
            flags: int = 0, counters: torch.Tensor = None, stream=None) -> torch.Tensor:
    """Sauvola binarization (Table 1): mask 0 = foreground."""
    H, W, pitch = _img2d(img)
    out = _alloc_mask(H, W, packed, img.device) if out is None else out
    _check(_lib.abin_sauvola(_ptr(img), H, W, pitch, _ptr(out), out.stride(0), MASK_BITS if packed else MASK_U8, h,
                             w, k, R, flags, _ptr(counters), _stream(stream)))
    return out


def niblack(img: torch.Tensor, h: int, w: int, k: float = -0.2, packed: bool = False, out=None, flags: int = 0,
            counters: torch.Tensor = None, stream=None) -> torch.Tensor:
    """Niblack binarization (Table 1)."""
    H, W, pitch = _img2d(img)
    out = _alloc_mask(H, W, packed, img.device) if out is None else out
    _check(_lib.abin_niblack(_ptr(img), H, W, pitch, _ptr(out), out.stride(0), MASK_BITS if packed else MASK_U8, h,
                             w, k, flags, _ptr(counters), _stream(stream)))
    return out


def wolf(img: torch.Tensor, h: int, w: int, k: float = 0.5, R: float = 128.0, L: int = -1, packed: bool = False,
         out=None, flags: int = 0, counters: torch.Tensor = None, stream=None) -> torch.Tensor:
    """Wolf binarization (Table 1); L < 0: global min on device."""
    H, W, pitch = _img2d(img)
    out = _alloc_mask(H, W, packed, img.device) if out is None else out
    _check(_lib.abin_wolf(_ptr(img), H, W, pitch, _ptr(out), out.stride(0), MASK_BITS if packed else MASK_U8, h, w, k,
                          R, L, flags, _ptr(counters), _stream(stream)))
    return out


def quantile(img: torch.Tensor, h: int, w: int, q: float = 0.5, packed: bool = False, out=None, flags: int = 0,
             stream=None) -> torch.Tensor:
    """Local-quantile threshold: mask 0 iff I <= Q."""
    H, W, pitch = _img2d(img)
    out = _alloc_mask(H, W, packed, img.device) if out is None else out
    _check(_lib.abin_quantile(_ptr(img), H, W, pitch, _ptr(out), out.stride(0), MASK_BITS if packed else MASK_U8, h,
                              w, q, flags, _stream(stream)))
    return out


def bernsen(img: torch.Tensor, h: int, w: int, contrast: int = -1, packed: bool = False, out=None, flags: int = 0,
            stream=None) -> torch.Tensor:
    """Bernsen midrange rule: mask 0 iff 2 I <= min + max of
    the window; contrast >= 0: 1 where max - min < contrast."""
    H, W, pitch = _img2d(img)
    out = _alloc_mask(H, W, packed, img.device) if out is None else out
    _check(_lib.abin_bernsen(_ptr(img), H, W, pitch, _ptr(out), out.stride(0), MASK_BITS if packed else MASK_U8, h,
                             w, contrast, flags, _stream(stream)))
    return out


def binarize_rule(rule: str, img: torch.Tensor, h: int, w: int, params=(), packed: bool = False, out=None,
                  flags: int = 0, counters: torch.Tensor = None, stream=None) -> torch.Tensor:
    """Feng / Rais / Khurshid / Phansalkar (Table 1); params as in abin.h."""
    H, W, pitch = _img2d(img)
    out = _alloc_mask(H, W, packed, img.device) if out is None else out
    prm = (ctypes.c_double * max(1, len(params)))(*params)
    _check(_lib.abin_binarize_rule(RULES[rule], _ptr(img), H, W, pitch, _ptr(out), out.stride(0),
                                   MASK_BITS if packed else MASK_U8, h, w, prm, len(params), flags, _ptr(counters),
                                   _stream(stream)))
    return out


def otsu(img: torch.Tensor, packed: bool = False, out=None, t_out: torch.Tensor = None, stream=None):
    """Otsu's global threshold: returns (mask, t) with t a device uint8 tensor."""
    H, W, pitch = _img2d(img)
    out = _alloc_mask(H, W, packed, img.device) if out is None else out
    t = torch.empty(1, dtype=torch.uint8, device=img.device) if t_out is None else t_out
    _check(_lib.abin_otsu(_ptr(img), H, W, pitch, _ptr(out), out.stride(0), MASK_BITS if packed else MASK_U8, _ptr(t),
                          0, _stream(stream)))
    return out, t


def binarize_batched(method: str, pages: torch.Tensor, h: int, w: int, param0: float, param1: float = 128.0,
                     L: int = -1, packed: bool = False, out=None, flags: int = 0, counters: torch.Tensor = None,
                     stream=None) -> torch.Tensor:
    """P pages (a (P, H, W) uint8 tensor, unit column stride) in one launch."""
    if pages.dtype != torch.uint8 or pages.dim() != 3 or pages.stride(2) != 1:
        raise ValueError("expected a (P, H, W) uint8 tensor with unit column stride")
    P, H, W = pages.shape
    if out is None:
        out = torch.empty((P, H, (W + 7) // 8 if packed else W), dtype=torch.uint8, device=pages.device)
    _check(_lib.abin_binarize_batched(METHODS[method], _ptr(pages), pages.stride(0), _ptr(out), out.stride(0), P, H,
                                      W, pages.stride(1), out.stride(1), MASK_BITS if packed else MASK_U8, h, w,
                                      param0, param1, L, flags, _ptr(counters), _stream(stream)))
    return out


def binarize_band(method: str, held: torch.Tensor, row0: int, H_global: int, halo_top: int, halo_bot: int, h: int,
                  w: int, param0: float, param1: float = 128.0, L: int = -1, packed: bool = False, out=None,
                  flags: int = 0, counters: torch.Tensor = None, stream=None) -> torch.Tensor:
    """Rows [row0, row0 + H_band) of an H_global-row image; `held` holds rows
    [row0 - halo_top, row0 + H_band + halo_bot)."""
    Hh, W, pitch = _img2d(held)
    H_band = Hh - halo_top - halo_bot
    out = _alloc_mask(H_band, W, packed, held.device) if out is None else out
    _check(_lib.abin_binarize_band(METHODS[method], _ptr(held), H_band, W, pitch, row0, H_global, halo_top, halo_bot,
                                   _ptr(out), out.stride(0), MASK_BITS if packed else MASK_U8, h, w, param0, param1, L,
                                   flags, _ptr(counters), _stream(stream)))
    return out


def global_min(pages: torch.Tensor, stream=None) -> torch.Tensor:
    """Per-page global minimum gray level L (Table 1 notation), on device."""
    if pages.dim() == 2:
        pages = pages.unsqueeze(0)
    P, H, W = pages.shape
    L = torch.empty(P, dtype=torch.uint8, device=pages.device)
    _check(_lib.abin_global_min(_ptr(pages), pages.stride(0), P, H, W, pages.stride(1), _ptr(L), _stream(stream)))
    return L


def max_s(img: torch.Tensor, h: int, w: int, row0: int = 0, H_global: int = None, halo_top: int = 0,
          halo_bot: int = 0, stream=None) -> float:
    """Max over the (band's own rows of the) image of the canonical s: Wolf's
    adaptive R source (R21).  `img` holds halo_top + own + halo_bot rows."""
    _img2d(img)
    Hb = img.shape[0] - halo_top - halo_bot
    out = ctypes.c_double()
    _check(_lib.abin_max_s(_ptr(img), Hb, img.shape[1], img.stride(0), row0, H_global if H_global else Hb,
                           halo_top, halo_bot, h, w, ctypes.byref(out), _stream(stream)))
    return out.value


def wolf_adaptive(img: torch.Tensor, h: int, w: int, k: float = 0.5, L: int = -1, packed: bool = False, out=None,
                  flags: int = 0, counters: torch.Tensor = None, stream=None):
    """Wolf with R = max s over the image (+inf if every window is constant);
    returns (mask, R).  One host synchronisation."""
    _img2d(img)
    H, W = img.shape
    if out is None:
        out = torch.empty((H, (W + 7) // 8 if packed else W), dtype=torch.uint8, device=img.device)
    R = ctypes.c_double()
    _check(_lib.abin_wolf_adaptive(_ptr(img), H, W, img.stride(0), _ptr(out), out.stride(0),
                                   MASK_BITS if packed else MASK_U8, h, w, k, L, flags, _ptr(counters),
                                   ctypes.byref(R), _stream(stream)))
    return out, R.value


def probe_filter(method: str, c: torch.Tensor, d: torch.Tensor, ncol: torch.Tensor, nrow: torch.Tensor,
                 I: torch.Tensor, k: float = 0.0, R: float = 128.0, L: float = 0.0, rule_params=None, stream=None):
    """Test hook: the kernel's fp32 residuals e~ = I - t~ (and s~) for tuples
    of exact window data (uint32 c, d, ncol, nrow; uint8 I, all on the device)
    and the certified bound [coarse, rb0, rb1, rdv, rsdv] (abin.h).  Rules
    "khurshid" / "phansalkar" take rule_params ({k, N_mode, h w} /
    {k, R, p, q})."""
    n = c.numel()
    e = torch.empty(n, dtype=torch.float32, device=c.device)
    sv = torch.empty(n, dtype=torch.float32, device=c.device)
    b = (ctypes.c_double * 5)()
    code = RULES[method] if method in RULES else METHODS[method]
    rp = None
    if rule_params is not None:
        rp = (ctypes.c_double * 5)(*([float(x) for x in rule_params] + [0.0] * (5 - len(rule_params))))
    _check(_lib.abin_probe_filter(code, k, R, L, rp, _ptr(c), _ptr(d), _ptr(ncol), _ptr(nrow), _ptr(I), n,
                                  _ptr(e), _ptr(sv), b, _stream(stream)))
    return e, sv, list(b)


def stats(method: str, img: torch.Tensor, h: int, w: int, param0: float, param1: float = 128.0, L: int = -1,
          stream=None) -> dict:
    """Per-pixel c, d (uint64), n (uint32), t (double; Q for quantile) and mask."""
    H, W, pitch = _img2d(img)
    dev = img.device
    c = torch.empty((H, W), dtype=torch.int64, device=dev)
    d = torch.empty((H, W), dtype=torch.int64, device=dev)
    n = torch.empty((H, W), dtype=torch.int32, device=dev)
    t = torch.empty((H, W), dtype=torch.float64, device=dev)
    m = torch.empty((H, W), dtype=torch.uint8, device=dev)
    quant = method in ("quantile", "bernsen")
    _check(_lib.abin_stats(METHODS[method], _ptr(img), H, W, pitch, h, w, param0, param1, L, None if quant else _ptr(c),
                           None if quant else _ptr(d), None if quant else _ptr(n), _ptr(t), _ptr(m), _stream(stream)))
    out = {"t": t, "mask": m}
    if not quant:
        out.update(c=c, d=d, n=n)
    return out


def strerror(status: int) -> str:
    return _lib.abin_strerror(status).decode()


def raw():
    """The ctypes handle (for the C-ABI conformance tests)."""
    return _lib
