"""GPU parity (-m gpu) of the packed last strips of the v5 moments kernel
(moments5.cuh PACK): in a page batch, the last (mostly empty) column strip of
NG pages runs in one warp.  Masks must equal the oracle's and the unpacked
launch's bit for bit: widths whose last strip holds 1 .. several output
lanes, window widths of 1 .. 8 halo lanes, batches that do and do not fill
the last pack, byte and bit masks, Wolf's per-page minimum, Niblack's exact
fixup entries from packed lanes, and the config-3 geometry (4960 columns)."""
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


def batch(P, H, W, seed):
    pages = synth.pages(P, H, W, synth.config_seed(9, seed), stain=True)
    pitch = (W + 15) // 16 * 16
    buf = torch.zeros((P, H, pitch), dtype=torch.uint8, device=DEV)
    buf[:, :, :W] = torch.from_numpy(pages).to(DEV)
    return pages, buf[:, :, :W]


# (pages, H, W, h, w): W = (n_strips - 1) Tw + remainder, Tw = 16 (32 - ceil(w / 16))
CASES = [(7, 70, 2 * 448 + 20, 61, 61), (5, 64, 448 + 32, 61, 61), (11, 40, 496 + 5, 9, 15),
         (6, 50, 2 * 480 + 40, 31, 31), (9, 33, 384 + 100, 21, 127), (4, 90, 4960, 61, 61),
         (3, 45, 448 + 1, 61, 60), (12, 20, 2 * 464 + 16, 5, 33)]


@pytest.mark.parametrize("case", CASES, ids=[f"P{c[0]}_{c[1]}x{c[2]}_w{c[3]}x{c[4]}" for c in CASES])
def test_packed_last_strips(monkeypatch, case):
    P, H, W, h, w = case
    pages, x = batch(P, H, W, P + W)
    for method in ("sauvola", "niblack", "wolf"):
        k, R = PARAMS[method]
        for packed in (False, True):
            monkeypatch.delenv("ABIN_NO_PACK", raising=False)
            got = ab.binarize_batched(method, x, h, w, k, R, packed=packed).cpu().numpy()
            monkeypatch.setenv("ABIN_NO_PACK", "1")
            ref_gpu = ab.binarize_batched(method, x, h, w, k, R, packed=packed).cpu().numpy()
            assert np.array_equal(got, ref_gpu), (method, packed)
            for p in range(P):
                ref = oracle.binarize(method, pages[p], h, w, k, R)
                assert np.array_equal(got[p], oracle.pack_bits(ref) if packed else ref), (method, packed, p)


def test_packed_niblack_fixup_entries():
    """Near-constant pages: packed lanes queue many ambiguous pixels for the
    exact fixup, which must patch the right page."""
    P, H, W = 6, 40, 448 + 24
    pages = np.full((P, H, W), 128, np.uint8)
    for p in range(P):
        pages[p, p::5, W - 17::3] = 130 + p
        pages[p, ::7, ::11] = 126
    x = torch.from_numpy(pages).to(DEV)
    got = ab.binarize_batched("niblack", x, 61, 61, -0.2, 128.0).cpu().numpy()
    for p in range(P):
        assert np.array_equal(got[p], oracle.binarize("niblack", pages[p], 61, 61, -0.2, 128.0)), p
