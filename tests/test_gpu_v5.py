"""GPU parity of the v5 moments kernel (moments5.cuh) -- -m gpu.

v5 is the production kernel for h <= 129, w <= 127 (uint32 square sums).  Its
horizontal pass reads the leaving columns at phase (-w) mod 16 and its own
columns at byte offset (w/2) mod 16 of the staged rows, both fixed at compile
time per w mod 32: every phase class is exercised here, on interior and border
strips, against the oracle (masks bit-exact, near-tie counts equal) and
against the v4 kernel (A/B through the ABIN_V4_INTERNAL test hook).
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
PARAMS = {"sauvola": (0.5, 128.0), "niblack": (-0.2, 128.0), "wolf": (0.5, 128.0)}


def to_dev(I):
    H, W = I.shape
    pitch = (W + 15) // 16 * 16
    buf = torch.zeros((H, pitch), dtype=torch.uint8, device=DEV)
    buf[:, :W] = torch.from_numpy(np.ascontiguousarray(I)).to(DEV)
    return buf[:, :W]


def run(method, x, h, w, flags=0, counters=None, packed=False):
    k, R = PARAMS[method]
    if method == "sauvola":
        return ab.sauvola(x, h, w, k, R, flags=flags, counters=counters, packed=packed)
    if method == "niblack":
        return ab.niblack(x, h, w, k, flags=flags, counters=counters, packed=packed)
    return ab.wolf(x, h, w, k, R, flags=flags, counters=counters, packed=packed)


def check(method, I, h, w, packed=False):
    k, R = PARAMS[method]
    st = oracle.binarize(method, I, h, w, k, R, stats=True)
    ref = st["mask"]
    x = to_dev(I)
    cnt = torch.zeros(2, dtype=torch.int64, device=DEV)
    got = run(method, x, h, w, counters=cnt, packed=packed).cpu().numpy()
    want = oracle.pack_bits(ref) if packed else ref
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{method} {I.shape} {h}x{w}: {len(bad)} mismatches, first {bad[:5].tolist()}"
    v4 = run(method, x, h, w, flags=abin.V4_INTERNAL, packed=packed).cpu().numpy()
    assert np.array_equal(got, v4)
    cnt = cnt.cpu().numpy()
    assert cnt[0] == st["near_tie"]
    return cnt


# every w mod 32 class (w = 1 .. 127 in steps that hit each class at least once)
W_ALL = list(range(1, 33)) + [45, 61, 64, 77, 95, 101, 113, 127]


@pytest.mark.parametrize("w", W_ALL)
def test_every_phase_sauvola(w):
    # 3 strips at w = 127 (Tw = 384): interior and both border variants
    I = synth.page(70, 1100, synth.config_seed(1, w), stain=True)
    check("sauvola", I, 15 if w > 2 else 3, w)


@pytest.mark.parametrize("method", ["niblack", "wolf"])
@pytest.mark.parametrize("w", [1, 2, 7, 16, 17, 31, 32, 33, 61, 64, 127])
def test_every_phase_other_rules(method, w):
    I = synth.page(60, 900, synth.config_seed(2, w), stain=True)
    check(method, I, 9, w)


@pytest.mark.parametrize("h", [1, 2, 3, 30, 61, 64, 100, 128, 129])
def test_window_heights(h):
    # top/bottom clipped rows (nrow < h), tall windows up to the v5 limit
    I = synth.page(150, 700, synth.config_seed(3, h), stain=True)
    check("sauvola", I, h, 61)
    check("niblack", I, h, 33)


@pytest.mark.parametrize("packed", [False, True])
def test_bit_mask_and_ragged_widths(packed):
    for W in (17, 449, 897, 1333):
        I = synth.page(40, W, synth.config_seed(4, W))
        check("sauvola", I, 11, 61, packed=packed)


def test_adversarial_near_ties():
    # low-contrast Niblack: thresholds within 1e-13 of the pixels -> the
    # certified filter queues these lanes and the exact fixup decides them
    rng = np.random.default_rng(5)
    I = (128 + rng.integers(-2, 3, size=(120, 800))).astype(np.uint8)
    cnt = check("niblack", I, 7, 7)
    assert cnt[1] > 0  # some pixels reached the exact stage
    C = np.full((64, 600), 77, np.uint8)
    cnt = check("niblack", C, 5, 9)           # constant: every pixel an exact tie
    assert cnt[0] == C.size
    check("sauvola", np.full((64, 600), 200, np.uint8), 5, 9)


def test_all_255_and_all_0_at_the_limits():
    for g in (0, 255):
        I = np.full((300, 600), g, np.uint8)
        I[::5, ::3] = 255 - g
        check("sauvola", I, 129, 127)
        check("wolf", I, 129, 127)


def test_batched_pages():
    P, H, W = 3, 200, 1000
    pages = synth.pages(P, H, W, synth.config_seed(3, 70), stain=True)
    x = torch.from_numpy(pages).to(DEV)
    out = ab.binarize_batched("sauvola", x, 61, 61, 0.5, 128.0)
    for p in range(P):
        assert np.array_equal(out[p].cpu().numpy(), oracle.binarize("sauvola", pages[p], 61, 61, 0.5, 128.0))



@pytest.mark.parametrize("W", [2550, 2553, 1000])
@pytest.mark.parametrize("hw", [9, 15])
@pytest.mark.parametrize("v4", [False, True])
def test_pad_columns_do_not_queue(W, hw, v4):
    """Columns past W in the last lane of a row lie wholly outside the image
    when w is small: their c = 0 gives t~ = 0 = I there.  They must not make
    the lane ambiguous.  On a constant page Sauvola's t = m (1 - k) is far
    from every pixel, so the exact fixup must see no pixel at all
    (ABIN_COUNT_STAGES counts them; before the fix every row queued its last
    lane), and the mask still equals the oracle's."""
    I = np.full((128, W), 200, np.uint8)
    x = to_dev(I)
    cnt = torch.zeros(3, dtype=torch.int64, device=DEV)
    flags = abin.COUNT_STAGES | (abin.V4_INTERNAL if v4 else 0)
    got = run("sauvola", x, hw, hw, flags=flags, counters=cnt).cpu().numpy()
    assert np.array_equal(got, oracle.binarize("sauvola", I, hw, hw, 0.5, 128.0))
    assert cnt.tolist() == [0, 0, 0]
