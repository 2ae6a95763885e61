"""Seeded random cases (-m gpu) for the round-2 paths, every mask against the
oracle bit for bit: the small-call kernel (single pages up to 2^22 pixels,
windows up to 64), the packed last strips of page batches (widths just past
a strip multiple, 2-7 pages), the window-independent Bernsen kernels, and
the Rais / Feng certified filters on random and document pages."""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1905_13038_b200 as ab  # noqa: E402

DEV = torch.device("cuda:0")
SCALE = int(os.environ.get("ABIN_FUZZ_SCALE", "1"))  # deeper one-off runs: more seeds per test
PARAMS = {"sauvola": (0.5, 128.0), "niblack": (-0.2, 128.0), "wolf": (0.5, 128.0)}


def _pages(rng, P, H, W, seed):
    kind = rng.integers(0, 3)
    if kind == 0:
        return rng.integers(0, 256, size=(P, H, W), dtype=np.uint8)
    if kind == 1:
        return synth.pages(P, H, W, synth.config_seed(11) + seed, stain=bool(seed & 1))
    pages = np.full((P, H, W), int(rng.integers(0, 256)), np.uint8)
    sel = rng.random((P, H, W)) < 0.02
    pages[sel] = rng.integers(0, 256, int(sel.sum()), dtype=np.uint8)
    return pages


def _device(pages, pad):
    P, H, W = pages.shape
    buf = torch.zeros((P, H, W + pad), dtype=torch.uint8, device=DEV)
    buf[:, :, :W] = torch.from_numpy(pages).to(DEV)
    return buf[:, :, :W]


@pytest.mark.small_path
@pytest.mark.parametrize("seed", range(40 * SCALE))
def test_fuzz_small_kernel(seed):
    rng = np.random.default_rng(1000 + seed)
    H, W = int(rng.integers(1, 300)), int(rng.integers(1, 700))
    h, w = int(rng.integers(1, 65)), int(rng.integers(1, 65))
    pages = _pages(rng, 1, H, W, seed)
    method = ["sauvola", "niblack", "wolf"][seed % 3]
    k, R = PARAMS[method]
    pad = int(rng.choice([0, 3, 16]))
    packed = bool(rng.integers(0, 2))
    got = ab.binarize_batched(method, _device(pages, pad), h, w, k, R, packed=packed).cpu().numpy()[0]
    ref = oracle.binarize(method, pages[0], h, w, k, R)
    assert np.array_equal(got, oracle.pack_bits(ref) if packed else ref), (seed, H, W, h, w, method, pad, packed)


@pytest.mark.parametrize("seed", range(24 * SCALE))
def test_fuzz_packed_strips(seed):
    rng = np.random.default_rng(2000 + seed)
    w = int(rng.integers(2, 128))
    KH = (w + 15) // 16
    Tw = 16 * (32 - KH)
    W = Tw * int(rng.integers(1, 3)) + int(rng.integers(1, 16 * max(1, 6 - KH) + 1))
    H, h = int(rng.integers(8, 60)), int(rng.integers(1, 60))
    P = int(rng.integers(2, 8))
    pages = _pages(rng, P, H, W, seed)
    method = ["sauvola", "niblack", "wolf"][seed % 3]
    k, R = PARAMS[method]
    packed = bool(rng.integers(0, 2))
    got = ab.binarize_batched(method, _device(pages, 0), h, w, k, R, packed=packed).cpu().numpy()
    for p in range(P):
        ref = oracle.binarize(method, pages[p], h, w, k, R)
        assert np.array_equal(got[p], oracle.pack_bits(ref) if packed else ref), (seed, p, W, h, w, method)


@pytest.mark.parametrize("seed", range(24 * SCALE))
def test_fuzz_bernsen(seed):
    rng = np.random.default_rng(3000 + seed)
    H, W = int(rng.integers(1, 200)), int(rng.integers(1, 600))
    h, w = int(rng.integers(1, 2 * H + 3)), int(rng.integers(1, min(2 * W + 3, 700)))
    P = int(rng.integers(1, 3))
    pages = _pages(rng, P, H, W, seed)
    contrast = int(rng.choice([-1, 0, 15, 60]))
    pad = int(rng.choice([0, 5, 16]))
    packed = bool(rng.integers(0, 2))
    got = ab.binarize_batched("bernsen", _device(pages, pad), h, w, float(contrast), packed=packed).cpu().numpy()
    for p in range(P):
        ref, _, _ = oracle.bernsen(pages[p], h, w, contrast)
        assert np.array_equal(got[p], oracle.pack_bits(ref) if packed else ref), (seed, p, H, W, h, w, contrast)


@pytest.mark.parametrize("seed", range(16 * SCALE))
def test_fuzz_rais_feng(seed):
    rng = np.random.default_rng(4000 + seed)
    H, W = int(rng.integers(20, 160)), int(rng.integers(20, 500))
    h, w = int(rng.integers(1, 100)), int(rng.integers(1, 100))
    pages = _pages(rng, 1, H, W, seed)
    x = _device(pages, 0)[0]
    if seed % 2:
        rule, prm = "rais", ()
    else:
        rule = "feng"
        prm = (float(rng.uniform(0.05, 0.3)), float(rng.uniform(0.0, 0.1)), float(rng.uniform(0.0, 0.05)),
               float(rng.choice([1.0, 1.5, 2.0, 3.0])), float(rng.choice([64.0, 128.0])))
    got = ab.binarize_rule(rule, x, h, w, prm).cpu().numpy()
    ref, t = oracle.binarize_rule(rule, pages[0], h, w, prm, with_t=True)
    if rule == "rais":
        assert np.array_equal(got, ref), (seed, H, W, h, w)
    else:  # Feng's pow: device vs glibc, near ties excluded (R18)
        tie = np.abs(pages[0].astype(np.float64) - t) < 1e-9
        assert not ((got != ref) & ~tie).any(), (seed, H, W, h, w, prm)
