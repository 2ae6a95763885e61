"""GPU parity (-m gpu) of the small-call kernel (csrc/small.cuh): single small
pages (here up to 2^22 pixels, windows up to 64 x 64) go to one launch of a
shared-memory tile kernel -- exact integer window sums, the certified fp32
residual and the canonical double threshold inline.  Masks and near-tie
counts must equal the oracle's bit for bit: odd / even windows, windows
reaching past the image, 1-row / 1-column pages, ragged tile edges, byte and
bit masks, tight and misaligned rows, the three rules, Niblack on near-
constant pages (every pixel through the double threshold), Wolf's minimum,
row bands, and the streaming kernels' masks on the same inputs."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.small_path]

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1905_13038_b200 as ab  # noqa: E402

DEV = torch.device("cuda:0")
PARAMS = {"sauvola": (0.5, 128.0), "niblack": (-0.2, 128.0), "wolf": (0.5, 128.0)}


def to_dev(I, pitch=None, offset=0):
    H, W = I.shape
    if pitch is None:
        pitch = (W + offset + 15) // 16 * 16
    buf = torch.zeros((H, pitch), dtype=torch.uint8, device=DEV)
    buf[:, offset:offset + W] = torch.from_numpy(np.ascontiguousarray(I)).to(DEV)
    return buf[:, offset:offset + W]


def run(method, x, h, w, packed=False, counters=None):
    k, R = PARAMS[method]
    if method == "sauvola":
        return ab.sauvola(x, h, w, k, R, packed=packed, counters=counters)
    if method == "niblack":
        return ab.niblack(x, h, w, k, packed=packed, counters=counters)
    return ab.wolf(x, h, w, k, R, packed=packed, counters=counters)


CASES = [((512, 512), (32, 32)), ((1, 1), (1, 1)), ((1, 300), (5, 5)), ((300, 1), (7, 3)), ((33, 129), (5, 6)),
         ((100, 257), (64, 64)), ((130, 700), (15, 15)), ((37, 41), (63, 64)), ((200, 300), (2, 1)),
         ((64, 128), (31, 33))]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0][0]}x{c[0][1]}_w{c[1][0]}x{c[1][1]}" for c in CASES])
def test_small_kernel_matches_oracle(case):
    (H, W), (h, w) = case
    I = synth.page(H, W, synth.config_seed(1, H + W), stain=True)
    for method in ("sauvola", "niblack", "wolf"):
        k, R = PARAMS[method]
        st = oracle.binarize(method, I, h, w, k, R, stats=True)
        ref = st["mask"]
        for pitch, offset in ((None, 0), (W, 0), (None, 5)):
            cnt = torch.zeros(2, dtype=torch.int64, device=DEV)
            got = run(method, to_dev(I, pitch, offset), h, w, counters=cnt).cpu().numpy()
            assert np.array_equal(got, ref), (method, pitch, offset)
            assert int(cnt[0]) == st["near_tie"], method
        got_b = run(method, to_dev(I), h, w, packed=True).cpu().numpy()
        assert np.array_equal(got_b, oracle.pack_bits(ref)), method


def test_small_kernel_near_constant_niblack():
    I = np.full((96, 200), 128, np.uint8)
    I[::7, ::5] = 131
    I[3::9, 1::4] = 125
    for h, w in ((9, 9), (40, 64)):
        st = oracle.binarize("niblack", I, h, w, -0.2, 128.0, stats=True)
        ref = st["mask"]
        cnt = torch.zeros(2, dtype=torch.int64, device=DEV)
        got = ab.niblack(to_dev(I), h, w, -0.2, counters=cnt).cpu().numpy()
        assert np.array_equal(got, ref)
        assert int(cnt[0]) == st["near_tie"]
    C = synth.constant(64, 64, 90)  # constant page: Niblack ties exactly everywhere
    assert np.array_equal(ab.niblack(to_dev(C), 5, 5, -0.2).cpu().numpy(), oracle.binarize("niblack", C, 5, 5, -0.2, 128.0))


def test_small_kernel_bands_and_streaming_twin(monkeypatch):
    J = synth.page(400, 350, synth.config_seed(1, 9))
    whole = oracle.binarize("sauvola", J, 31, 25, 0.5, 128.0)
    for G in (2, 3):
        bounds = np.linspace(0, 400, G + 1).astype(int)
        parts = []
        for g in range(G):
            r0, r1 = bounds[g], bounds[g + 1]
            top, bot = min(15, r0), min(15, 400 - r1)
            held = to_dev(np.ascontiguousarray(J[r0 - top:r1 + bot]))
            parts.append(ab.binarize_band("sauvola", held, r0, 400, top, bot, 31, 25, 0.5, 128.0).cpu().numpy())
        assert np.array_equal(np.concatenate(parts), whole)
    x = to_dev(J)
    a = ab.sauvola(x, 31, 25).cpu().numpy()
    monkeypatch.setenv("ABIN_SMALL_PX", "0")
    b = ab.sauvola(x, 31, 25).cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(a, whole)


def test_small_kernel_megapixel_page(monkeypatch):
    # the size limit is 2^22 pixels: a
    # ragged 1.43 Mpx page (9 x 69 tiles + partial tiles) against the oracle and
    # the streaming kernels, byte and bit masks
    J = synth.page(1100, 1301, synth.config_seed(2, 3))
    x = to_dev(J)
    for (h, w) in ((32, 32), (15, 17)):
        ref = oracle.binarize("sauvola", J, h, w, 0.5, 128.0)
        a = ab.sauvola(x, h, w).cpu().numpy()
        ab_bits = ab.sauvola(x, h, w, packed=True).cpu().numpy()
        monkeypatch.setenv("ABIN_SMALL_PX", "0")
        b = ab.sauvola(x, h, w).cpu().numpy()
        monkeypatch.delenv("ABIN_SMALL_PX")
        assert np.array_equal(a, ref) and np.array_equal(b, ref), (h, w)
        assert np.array_equal(ab_bits, oracle.pack_bits(ref)), (h, w)
    # 61 x 61 (Wolf: the page minimum from the device) on the same page and on its first 800 rows
    ref = oracle.binarize("wolf", J, 61, 61, 0.5, 128.0)
    assert np.array_equal(ab.wolf(x, 61, 61, 0.5, 128.0).cpu().numpy(), ref)
    K = np.ascontiguousarray(J[:800])
    assert np.array_equal(ab.wolf(to_dev(K), 61, 61, 0.5, 128.0).cpu().numpy(), oracle.binarize("wolf", K, 61, 61, 0.5, 128.0))
    # near the 2^22-pixel limit: the tile kernel's masks equal the streaming kernels'
    # (themselves pinned to the oracle at full size in test_gpu_fullsize.py)
    B = to_dev(synth.page(2040, 2050, synth.config_seed(2, 4)))
    for (h, w, packed) in ((15, 15, False), (33, 64, True)):
        a = ab.niblack(B, h, w, -0.2, packed=packed).cpu().numpy()
        monkeypatch.setenv("ABIN_SMALL_PX", "0")
        b = ab.niblack(B, h, w, -0.2, packed=packed).cpu().numpy()
        monkeypatch.delenv("ABIN_SMALL_PX")
        assert np.array_equal(a, b), (h, w)


def test_small_kernel_tall_tiles(monkeypatch):
    # 32-row tiles (taken when 16-row tiles would number more than 8 per SM;
    # ABIN_SMALL_TH32=0 forces them): ragged page heights around the tile
    # height, the three rules, byte and bit masks, against the oracle
    monkeypatch.setenv("ABIN_SMALL_TH32", "0")
    for (H, W, h, w) in ((33, 130, 5, 7), (95, 257, 32, 32), (64, 128, 64, 64), (1, 300, 9, 3)):
        I = synth.page(H, W, synth.config_seed(1, H))
        x = to_dev(I)
        for method in ("sauvola", "niblack", "wolf"):
            k, R = PARAMS[method]
            ref = oracle.binarize(method, I, h, w, k, R)
            assert np.array_equal(run(method, x, h, w).cpu().numpy(), ref), (method, H, W, h, w)
            assert np.array_equal(run(method, x, h, w, packed=True).cpu().numpy(), oracle.pack_bits(ref)), (method, H, W)
