"""C-ABI conformance on CPU (-m "not gpu"): libabin.so loads, exports every
symbol include/abin.h declares, and rejects bad arguments before touching a
device (no compute calls are made here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1905_13038_b200 import build
    build.build()
    from paper_1905_13038_b200 import abin
    return abin


def header_symbols():
    src = open(os.path.join(ROOT, "include", "abin.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(abin_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    syms = header_symbols()
    for name in ("abin_sauvola", "abin_niblack", "abin_wolf", "abin_quantile"):
        assert name in syms


def test_library_exports_every_header_symbol(lib):
    raw = lib.raw()
    for name in header_symbols():
        assert hasattr(raw, name), name
    assert set(lib.EXPORTED) == set(header_symbols())


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(ROOT, "paper_1905_13038_b200", "libabin.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_version_and_strerror(lib):
    assert "abin" in lib.version()
    for code in range(6):
        assert lib.strerror(code)
    assert lib.limits().max_window_w > 1000


FAKE_IN = 0x10000000
FAKE_OUT = 0x20000000


def call_sauvola(lib, **kw):
    a = dict(inp=FAKE_IN, H=64, W=64, pitch=64, out=FAKE_OUT, opitch=64, fmt=0, h=15, w=15, k=0.5, R=128.0)
    a.update(kw)
    return lib.raw().abin_sauvola(a["inp"], a["H"], a["W"], a["pitch"], a["out"], a["opitch"], a["fmt"], a["h"],
                                  a["w"], a["k"], a["R"], 0, None, None)


@pytest.mark.parametrize("kw,code", [
    (dict(inp=None), 1), (dict(out=None), 1), (dict(H=0), 1), (dict(W=0), 1), (dict(h=0), 1), (dict(w=-3), 1),
    (dict(pitch=63), 1), (dict(opitch=10), 1), (dict(fmt=7), 1), (dict(R=0.0), 1), (dict(R=-1.0), 1),
    (dict(k=float("nan")), 1), (dict(k=float("inf")), 1), (dict(R=float("nan")), 1),
    (dict(out=FAKE_IN + 100), 2), (dict(inp=FAKE_OUT - 10), 2),
])
def test_validation_errors(lib, kw, code):
    assert call_sauvola(lib, **kw) == code


def test_bits_format_pitch_rule(lib):
    # ceil(W/8) bytes per row suffice for ABIN_MASK_BITS
    assert call_sauvola(lib, fmt=1, opitch=7) == 1
    raw = lib.raw()
    # quantile q must lie in (0, 1]
    for q in (0.0, -0.1, 1.5, float("nan")):
        assert raw.abin_quantile(FAKE_IN, 8, 8, 8, FAKE_OUT, 8, 0, 3, 3, q, 0, None) == 1


def test_band_validation(lib):
    raw = lib.raw()
    # h = 11 -> o = 6, u = 5: a middle band needs 5 rows above and 5 below
    args = lambda top, bot, row0=100, Hb=50, Hg=400: raw.abin_binarize_band(
        0, FAKE_IN, Hb, 64, 64, row0, Hg, top, bot, FAKE_OUT, 64, 0, 11, 11, 0.5, 128.0, -1, 0, None, None)
    assert args(4, 5) == 1
    assert args(5, 4) == 1
    assert args(5, 5, row0=0) == 1            # halo above the image
    # a first band needs no rows above the image: validation accepts it (with
    # no CUDA device the first runtime call then fails with ABIN_ECUDA; on a
    # GPU box the fake pointers must not reach a kernel, so it is not called)
    import torch
    if not torch.cuda.is_available():
        assert args(0, 5, row0=0, Hg=400) == 4
    # Wolf bands need the global L
    assert raw.abin_binarize_band(2, FAKE_IN, 50, 64, 64, 100, 400, 5, 5, FAKE_OUT, 64, 0, 11, 11, 0.5, 128.0, -1,
                                  0, None, None) == 1


def test_batched_validation(lib):
    raw = lib.raw()
    # page stride smaller than a page
    assert raw.abin_binarize_batched(0, FAKE_IN, 100, FAKE_OUT, 64 * 64, 2, 64, 64, 64, 64, 0, 5, 5, 0.5, 128.0, -1,
                                     0, None, None) == 1
    # unknown method
    assert raw.abin_binarize_batched(9, FAKE_IN, 4096, FAKE_OUT, 4096, 1, 64, 64, 64, 64, 0, 5, 5, 0.5, 128.0, -1,
                                     0, None, None) == 1
    # overlapping page ranges
    assert raw.abin_binarize_batched(0, FAKE_IN, 4096, FAKE_IN + 4096 * 3, 4096, 4, 64, 64, 64, 64, 0, 5, 5, 0.5,
                                     128.0, -1, 0, None, None) == 2


def test_product_path_does_not_touch_the_oracle():
    # The product package must not import, link or execute anything under oracle/.
    pkg = os.path.join(ROOT, "paper_1905_13038_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, flags=re.M), f
                assert "liboracle" not in txt and "abin_oracle" not in txt, f


def test_limits_match_the_erange_checks(lib):
    """abin_limits states what each path takes; one step beyond returns
    ABIN_ERANGE before the device is touched (no compute call is made)."""
    raw = lib.raw()
    L = lib.limits()
    assert L.max_dim == 1 << 30
    assert L.max_window_hw == ((1 << 32) - 1) // 255
    assert L.quantile_max_window_w == 385 and L.quantile_max_window_hw == 65535
    H = W = 1000
    q = lambda h, w: raw.abin_binarize_batched(3, FAKE_IN, H * W, FAKE_OUT, H * W, 1, H, W, W, W, 0, h, w, 0.5, 0.0,
                                               -1, 0, None, None)
    assert q(3, L.quantile_max_window_w + 1) == 3            # quantile width
    assert q(256, 256) == 3                                  # h w > 65535
    b = lambda h, w: raw.abin_binarize_batched(4, FAKE_IN, H * W, FAKE_OUT, H * W, 1, H, W, W, W, 0, h, w, -1.0, 0.0,
                                               -1, 0, None, None)
    assert L.bernsen_max_window_w == 2048
    big = 1 << 20
    bb = lambda h, w: raw.abin_binarize_batched(4, FAKE_IN, big, FAKE_OUT, big, 1, 8, big, big, big, 0, h, w, -1.0,
                                                0.0, -1, 0, None, None)
    assert bb(3, L.bernsen_max_window_w + 1) == 3            # Bernsen: the row pass's staged tile
    # moments: effective sizes are clamped to the image, so a huge window on a
    # big (fake) image exceeds the width limit
    m = lambda h, w: raw.abin_binarize_batched(0, FAKE_IN, big, FAKE_OUT, big, 1, 8, big, big, big, 0, h, w, 0.5,
                                               128.0, -1, 0, None, None)
    assert m(3, L.max_window_w + 1) == 3


def test_table1_rules_only_through_binarize_rule(lib):
    # methods 5..8 need their parameter array: the batched / band / stats
    # entry points reject them
    raw = lib.raw()
    for method in (5, 6, 7, 8):
        assert raw.abin_binarize_batched(method, FAKE_IN, 4096, FAKE_OUT, 4096, 1, 64, 64, 64, 64, 0, 5, 5, 0.5,
                                         128.0, -1, 0, None, None) == 1
        assert raw.abin_binarize_band(method, FAKE_IN, 50, 64, 64, 100, 400, 5, 5, FAKE_OUT, 64, 0, 11, 11, 0.5,
                                      128.0, 7, 0, None, None) == 1
        assert raw.abin_stats(method, FAKE_IN, 64, 64, 64, 5, 5, 0.5, 128.0, -1, None, None, None, None, None,
                              None) == 1
