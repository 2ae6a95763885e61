"""GPU parity (-m gpu) of the window-independent Bernsen kernels
(csrc/bernsen.cuh: van Herk / Gil-Werman row and column passes) against the
direct-extrema oracle (oracle/abin_oracle.c orc_bernsen), bit
for bit: window sizes on both sides of the row tile (128 / 256 outputs) and
of the image, odd / even sizes, 1-pixel images and windows, heights beyond
the histogram kernels' reach, ragged widths, padded / tight / misaligned
rows, byte and bit masks, the local-contrast variant, page batches, row bands
with halos, and agreement with the histogram kernels (Q2_INTERNAL)."""
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


def to_dev(I, pitch=None, offset=0):
    """(H, W) page on the device; pitch None: 16-byte padded rows; offset:
    the first column sits `offset` bytes into its row (a misaligned base)."""
    H, W = I.shape
    if pitch is None:
        pitch = (W + offset + 15) // 16 * 16
    buf = torch.zeros((H, pitch), dtype=torch.uint8, device=DEV)
    buf[:, offset:offset + W] = torch.from_numpy(np.ascontiguousarray(I)).to(DEV)
    return buf[:, offset:offset + W]


def image(kind, H, W, seed):
    rng = np.random.default_rng(seed)
    if kind == "random":
        return rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    if kind == "levels":  # few levels: many ties of min / max and of 2 I = min + max
        return (rng.integers(0, 4, size=(H, W)) * 85).astype(np.uint8)
    return synth.page(H, W, synth.config_seed(7, seed), stain=True)


CASES = [  # (H, W), (h, w)
    ((1, 1), (1, 1)), ((1, 1), (5, 5)), ((1, 300), (3, 7)), ((300, 1), (7, 3)), ((33, 41), (5, 5)),
    ((64, 200), (51, 51)), ((7, 300), (4, 9)), ((100, 3), (3, 100)), ((130, 257), (16, 31)),
    ((90, 333), (1, 127)), ((90, 333), (2, 128)), ((77, 290), (9, 129)), ((61, 700), (3, 255)),
    ((61, 700), (6, 256)), ((40, 900), (5, 300)), ((50, 600), (1, 1)), ((300, 50), (301, 3)),
    ((260, 70), (199, 12)), ((45, 45), (90, 90)),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0][0]}x{c[0][1]}_w{c[1][0]}x{c[1][1]}" for c in CASES])
def test_bernsen_vh_matches_oracle(case):
    (H, W), (h, w) = case
    for kind in ("random", "levels", "page"):
        I = image(kind, H, W, H * 7 + W + h)
        for contrast in (-1, 0, 20, 256):
            ref, _, _ = oracle.bernsen(I, h, w, contrast)
            for pitch, offset in ((None, 0), (W, 0), (None, 3)):
                x = to_dev(I, pitch, offset)
                got = ab.bernsen(x, h, w, contrast).cpu().numpy()
                assert np.array_equal(got, ref), (kind, contrast, pitch, offset)
            got_b = ab.bernsen(to_dev(I), h, w, contrast, packed=True).cpu().numpy()
            assert np.array_equal(got_b, oracle.pack_bits(ref)), (kind, contrast)


def test_bernsen_vh_equals_histogram_kernels():
    """The new path and the round-1 sliding-histogram kernels give the same
    masks (two independent GPU implementations of the same definition)."""
    for (H, W), (h, w) in [((200, 500), (51, 51)), ((129, 385), (21, 64)), ((64, 1000), (15, 15))]:
        I = image("page", H, W, h + w)
        x = to_dev(I)
        for contrast in (-1, 15):
            a = ab.bernsen(x, h, w, contrast).cpu().numpy()
            b = ab.bernsen(x, h, w, contrast, flags=abin.Q2_INTERNAL).cpu().numpy()
            assert np.array_equal(a, b)


def test_bernsen_vh_large_windows_sampled():
    """Windows far beyond the histogram kernels' limits (h w > 65535, w > 385)
    on a 1000 x 1400 page: sampled pixels (every border row and column, the
    tile seams, random interior) against the oracle evaluated point by point."""
    H, W = 1000, 1400
    I = image("page", H, W, 5)
    x = to_dev(I)
    rng = np.random.default_rng(11)
    for h, w, n in ((301, 301, 20000), (255, 1000, 8000), (999, 17, 20000), (2001, 2001, 300)):
        m = ab.bernsen(x, h, w, 10).cpu().numpy()
        edge = [0, H - 1] if n < 1000 else [0, 1, H // 2, H - 2, H - 1]
        rows = np.concatenate([np.repeat(edge, W), rng.integers(0, H, n)])
        cols = np.concatenate([np.tile(np.arange(W), len(edge)), rng.integers(0, W, n)])
        seam = np.arange(0, W, 128)
        srows = np.arange(0, H, 7 if n >= 1000 else 97)
        rows = np.concatenate([rows, np.repeat(srows, seam.size)])
        cols = np.concatenate([cols, np.tile(seam, srows.size)])
        ref = oracle.bernsen_points(I, h, w, 10, rows, cols)
        assert np.array_equal(m[rows, cols], ref), (h, w)


def test_bernsen_vh_batches_and_bands():
    P = synth.pages(4, 150, 333, synth.config_seed(7, 3))
    for packed in (False, True):
        mb = ab.binarize_batched("bernsen", torch.from_numpy(P).to(DEV), 31, 45, 12.0, packed=packed).cpu().numpy()
        for p in range(4):
            ref = oracle.bernsen(P[p], 31, 45, 12)[0]
            assert np.array_equal(mb[p], oracle.pack_bits(ref) if packed else ref)
    J = synth.page(700, 410, synth.config_seed(7, 4))
    for h in (41, 40):
        whole, _, _ = oracle.bernsen(J, h, 33, -1)
        o, u = (h + 1) // 2, h // 2
        for G in (2, 3, 7):
            bounds = np.linspace(0, 700, G + 1).astype(int)
            parts = []
            for g in range(G):
                r0, r1 = bounds[g], bounds[g + 1]
                top, bot = min(o - 1, r0), min(u, 700 - r1)
                held = to_dev(np.ascontiguousarray(J[r0 - top:r1 + bot]))
                parts.append(ab.binarize_band("bernsen", held, r0, 700, top, bot, h, 33, -1.0).cpu().numpy())
            assert np.array_equal(np.concatenate(parts), whole), (h, G)
