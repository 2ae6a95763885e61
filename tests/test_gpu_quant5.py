"""GPU parity of the v5 quantile kernel (quantile5.cuh) -- -m gpu.

v5 decides I <= Q through the window count #(x < I) kept at 16-level CDF
windows, with an exact queue for the pixels no window decides (DESIGN.md
section 5, K5).  Its address arithmetic is fixed at compile time per
w mod 16 (the leaving column's lane and slot), so every class is checked here
against the oracle (masks bit-exact) and against the round-1 kernels (A/B via
the ABIN_Q2_INTERNAL test hook); the exact queue is exercised by forcing
windows that decide nothing (ABIN_Q5_FORCE_L), and its inline overflow path
by a one-entry queue (ABIN_Q5_QCAP).
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1905_13038_b200 as ab  # noqa: E402
from paper_1905_13038_b200 import abin  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(autouse=True)
def _v5_for_every_q(monkeypatch):
    # the library keeps q < 0.25 on the round-1 kernels; here v5 takes every q
    monkeypatch.setenv("ABIN_Q5_ALWAYS", "1")


def to_dev(I):
    H, W = I.shape
    pitch = (W + 15) // 16 * 16
    buf = torch.zeros((H, pitch), dtype=torch.uint8, device=DEV)
    buf[:, :W] = torch.from_numpy(np.ascontiguousarray(I)).to(DEV)
    return buf[:, :W]


def run(I, h, w, q, packed=False, flags=0, aligned=True):
    """One page through binarize_batched: 16-byte aligned input and mask rows
    (v5's vector loads / stores), or tight rows (its byte-wise path)."""
    H, W = I.shape
    x = to_dev(I) if aligned else torch.from_numpy(np.ascontiguousarray(I)).to(DEV)
    ow = (W + 7) // 8 if packed else W
    opitch = (ow + 15) // 16 * 16 if aligned else ow
    out = torch.zeros((1, H, opitch), dtype=torch.uint8, device=DEV)[:, :, :ow]
    cnt = torch.zeros(3, dtype=torch.int64, device=DEV)
    ab.binarize_batched("quantile", _as_batch(x), h, w, q, packed=packed, flags=flags, counters=cnt, out=out)
    return out[0].cpu().numpy(), int(cnt[1])


def _as_batch(x):
    # a (1, H, W) view of a pitched 2-D tensor
    return x.as_strided((1, x.shape[0], x.shape[1]), (x.shape[0] * x.stride(0), x.stride(0), 1))


def check(I, h, w, q, packed=False, tight=True):
    ref, _ = oracle.quantile(I, h, w, q)
    want = oracle.pack_bits(ref) if packed else ref
    got, n_exact = run(I, h, w, q, packed)
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{I.shape} {h}x{w} q={q}: {len(bad)} mismatches, first {bad[:5].tolist()}"
    if tight:
        got_t, _ = run(I, h, w, q, packed, aligned=False)
        assert np.array_equal(got_t, want), "byte-wise path"
    old, _ = run(I, h, w, q, packed, flags=abin.Q2_INTERNAL)
    assert np.array_equal(got, old)
    return n_exact


W_ALL = list(range(1, 33)) + [45, 51, 61, 64, 77, 101, 113, 127]


@pytest.mark.parametrize("w", W_ALL)
def test_every_phase(w):
    # 3 strips at w = 127 (Tw = 256): interior and both border variants
    I = synth.page(60, 1100, synth.config_seed(5, w))
    for q in (0.5, 0.1):
        check(I, 15 if w > 2 else 3, w, q)


@pytest.mark.parametrize("h", [1, 2, 3, 30, 64, 129, 200, 255])
def test_window_heights(h):
    I = synth.page(300, 700, synth.config_seed(6, h))
    check(I, h, 51, 0.5)
    check(I, h, 17, 0.9)


@pytest.mark.parametrize("q", [0.5, 0.1, 0.9, 1.0, 0.001, 0.37])
def test_document_page_and_extremes(q):
    I = synth.page(260, 1500, synth.config_seed(5, 7))
    check(I, 51, 51, q)


@pytest.mark.parametrize("packed", [False, True])
def test_ragged_widths_and_bits(packed):
    for W in (1, 17, 449, 450, 897, 1333):
        I = synth.page(40, W, synth.config_seed(5, W))
        check(I, 11, 51, 0.5, packed=packed)
        check(I, 5, 3, 0.1, packed=packed)


def test_uniform_noise_and_constant_pages():
    rng = np.random.default_rng(9)
    I = rng.integers(0, 256, size=(200, 900), dtype=np.uint8)   # Q spread over all levels
    for q in (0.5, 0.1, 0.9):
        check(I, 51, 51, q)
    for g in (0, 255, 77):
        check(np.full((64, 600), g, np.uint8), 9, 9, 0.5)


@pytest.mark.parametrize("force_L,qcap", [(0, None), (240, None), (100, "1"), (0, "37")])
def test_exact_queue_and_inline_overflow(monkeypatch, force_L, qcap):
    """Windows forced away from the data decide (almost) nothing: the exact
    queue, and with a tiny queue the inline path, must give the same mask."""
    monkeypatch.setenv("ABIN_Q5_FORCE_L", str(force_L))
    if qcap:
        monkeypatch.setenv("ABIN_Q5_QCAP", qcap)
    I = synth.page(90, 700, synth.config_seed(5, 11))
    for q, packed in ((0.5, False), (0.1, True)):
        n_exact = check(I, 21, 33, q, packed=packed)
        assert n_exact > 0


def test_batch_and_windows(monkeypatch):
    pages = synth.pages(3, 150, 777, synth.config_seed(5, 12))
    buf = torch.zeros((3, 150, 784), dtype=torch.uint8, device=DEV)   # 16-byte aligned rows (v5's loads)
    buf[:, :, :777] = torch.from_numpy(pages).to(DEV)
    x = buf[:, :, :777]
    for nw in ("1", "2", "3"):
        monkeypatch.setenv("ABIN_Q5_NW", nw)
        for q in (0.5, 0.1):
            out = ab.binarize_batched("quantile", x, 51, 51, q).cpu().numpy()
            for p in range(3):
                assert np.array_equal(out[p], oracle.quantile(pages[p], 51, 51, q)[0]), (nw, q, p)


def test_exact_decisions_are_rare_on_document_pages():
    """The windows placed from the tile sample leave few pixels to the exact
    queue on the config-5 recipe (a performance property; the masks are exact
    either way)."""
    I = synth.page(256, 4096, synth.config_seed(5))   # config 5's width (its gradient per strip)
    for q, bound in ((0.5, 1e-3), (0.9, 1e-3)):
        n = check(I, 51, 51, q)
        assert n <= bound * I.size, (q, n)
