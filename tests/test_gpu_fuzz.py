"""Seeded random cases (-m gpu): shapes, windows, pitches, page batches, mask
formats and methods drawn at random, every mask checked against the oracle
bit for bit.  The cases are small (the oracle is the direct definition) but
cover what the fixed tests pin one at a time: the re-pitch of unaligned rows,
the fixup queue sized to the call, the paired histogram kernel's odd widths
and both quantile walk modes, windows larger than the image."""
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
PARAMS = {"sauvola": (0.5, 128.0), "niblack": (-0.2, 128.0), "wolf": (0.5, 128.0)}


def _case(seed):
    rng = np.random.default_rng(seed)
    H = int(rng.integers(1, 110))
    W = int(rng.integers(1, 260))
    h = int(rng.integers(1, min(2 * H + 3, 121)))
    w = int(rng.integers(1, min(2 * W + 3, 121)))
    P = int(rng.integers(1, 4))
    kind = rng.integers(0, 3)
    if kind == 0:
        pages = rng.integers(0, 256, size=(P, H, W), dtype=np.uint8)
    elif kind == 1:
        pages = synth.pages(P, H, W, synth.config_seed(3) + seed, stain=bool(seed & 1))
    else:  # near-flat pages: Niblack ties, long quantile walks
        pages = np.full((P, H, W), int(rng.integers(0, 256)), np.uint8)
        sel = rng.random((P, H, W)) < 0.01
        pages[sel] = rng.integers(0, 256, int(sel.sum()), dtype=np.uint8)
    pad = int(rng.choice([0, 0, 1, 5, 16]))
    packed = bool(rng.integers(0, 2))
    return pages, h, w, pad, packed, rng


def _device(pages, pad):
    P, H, W = pages.shape
    buf = torch.zeros((P, H, W + pad), dtype=torch.uint8, device=DEV)
    buf[:, :, :W] = torch.from_numpy(pages).to(DEV)
    return buf[:, :, :W]


@pytest.mark.parametrize("seed", range(96))
def test_fuzz_moments(seed):
    pages, h, w, pad, packed, rng = _case(seed)
    method = ["sauvola", "niblack", "wolf"][seed % 3]
    k, R = PARAMS[method]
    x = _device(pages, pad)
    got = ab.binarize_batched(method, x, h, w, k, R, packed=packed).cpu().numpy()
    for p in range(pages.shape[0]):
        ref = oracle.binarize(method, pages[p], h, w, k, R)
        want = oracle.pack_bits(ref) if packed else ref
        assert np.array_equal(got[p], want), (seed, method, pages.shape, h, w, pad, packed, p)


@pytest.mark.parametrize("seed", range(64))
def test_fuzz_quantile_bernsen(seed):
    pages, h, w, pad, packed, rng = _case(1000 + seed)
    pages = pages[:, :90, :200]  # the sort-based oracle is slower
    h, w = min(h, 41), min(w, 41)
    x = _device(np.ascontiguousarray(pages), pad)
    if seed % 2 == 0:
        q = float(rng.choice([0.05, 0.1, 0.3, 0.5, 0.9, 1.0]))
        got = ab.binarize_batched("quantile", x, h, w, q, packed=packed).cpu().numpy()
        for p in range(pages.shape[0]):
            ref, _ = oracle.quantile(np.ascontiguousarray(pages[p]), h, w, q)
            want = oracle.pack_bits(ref) if packed else ref
            assert np.array_equal(got[p], want), (seed, q, pages.shape, h, w, pad, packed, p)
    else:
        contrast = int(rng.choice([-1, 10, 40]))
        got = ab.binarize_batched("bernsen", x, h, w, float(contrast), packed=packed).cpu().numpy()
        for p in range(pages.shape[0]):
            ref, _, _ = oracle.bernsen(np.ascontiguousarray(pages[p]), h, w, contrast)
            want = oracle.pack_bits(ref) if packed else ref
            assert np.array_equal(got[p], want), (seed, contrast, pages.shape, h, w, pad, packed, p)


@pytest.mark.parametrize("seed", range(32))
def test_fuzz_otsu(seed):
    """Otsu: the block-parallel split scan picks the oracle's t,
    including ties (two- and three-level images make the between-class
    variance equal over whole ranges of t: the smallest t must win)."""
    rng = np.random.default_rng(5000 + seed)
    H, W = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    kind = seed % 4
    if kind == 0:
        I = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    elif kind == 1:
        levels = rng.choice(256, size=int(rng.integers(1, 4)), replace=False).astype(np.uint8)
        I = levels[rng.integers(0, levels.size, size=(H, W))]
    elif kind == 2:
        I = synth.page(max(H, 8), max(W, 8), synth.config_seed(9) + seed, stain=True)
    else:
        I = np.clip(rng.normal(128, 40, size=(H, W)), 0, 255).astype(np.uint8)
    t, ref = oracle.otsu(I)
    pad = int(rng.choice([0, 3, 16]))
    buf = torch.zeros((I.shape[0], I.shape[1] + pad), dtype=torch.uint8, device=DEV)
    buf[:, :I.shape[1]] = torch.from_numpy(np.ascontiguousarray(I)).to(DEV)
    m, tt = ab.otsu(buf[:, :I.shape[1]])
    assert int(tt.item()) == t, (seed, kind, I.shape)
    assert np.array_equal(m.cpu().numpy(), ref)
