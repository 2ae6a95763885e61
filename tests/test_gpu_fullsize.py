"""Full-size parity (-m gpu): every BASELINE.json config at its full size, in
the launch configuration bench.py times, checked against the oracle on
sampled pixels (the oracle evaluates the paper's definition pixel by pixel,
oracle.binarize_points / quantile_points) plus properties that hold at any
size.  Samples cover every image edge and corner, the seams between the
kernel's warp strips (every 448 / 432 columns for w = 61 / 101) and row
bands, and uniform random pixels.  Bars as in test_gpu_parity.py: masks bit-
exact; near ties counted (zero expected on these pages)."""
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
from paper_1905_13038_b200 import dist as adist  # noqa: E402

DEV = torch.device("cuda:0")


def sample_points(H, W, n_random, seed, seam=448):
    """Edges, corners, strip seams (+-2 columns around every multiple of the
    warp-strip width) and uniform random pixels."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for r in (0, 1, 2, H // 2, H - 3, H - 2, H - 1):          # full rows at the top / middle / bottom
        c = np.arange(0, W, max(1, W // 997))
        rows.append(np.full(c.size, r)); cols.append(c)
    for c in (0, 1, W // 2, W - 2, W - 1):                      # full columns at the edges
        r = np.arange(0, H, max(1, H // 997))
        rows.append(r); cols.append(np.full(r.size, c))
    seams = np.concatenate([np.arange(s - 2, s + 3) for s in range(seam, W, seam)]) if W > seam else np.array([], int)
    if seams.size:
        r = rng.integers(0, H, seams.size * 8)
        rows.append(r); cols.append(np.repeat(seams, 8))
    rows.append(rng.integers(0, H, n_random)); cols.append(rng.integers(0, W, n_random))
    rows = np.concatenate(rows).astype(np.int64)
    cols = np.concatenate(cols).astype(np.int64)
    keep = (cols >= 0) & (cols < W) & (rows >= 0) & (rows < H)
    return rows[keep], cols[keep]


def device_pages(P, H, W, cfg, stain):
    host = synth.pages(P, H, W, synth.config_seed(cfg), stain=stain)
    pitch = (W + 15) // 16 * 16
    buf = torch.zeros((P, H, pitch), dtype=torch.uint8, device=DEV)
    buf[:, :, :W] = torch.from_numpy(host).to(DEV)
    return host, buf[:, :, :W]


def unpack(bits, W):
    return np.unpackbits(bits, axis=-1, bitorder="big")[..., :W]


@pytest.fixture(scope="module")
def config3():
    return device_pages(64, 7016, 4960, 3, True)


@pytest.mark.parametrize("method,k", [("sauvola", 0.5), ("niblack", -0.2), ("wolf", 0.5)])
def test_config3_64_pages_sampled(config3, method, k):
    """Config 3: 64 pages of 7016 x 4960 + stain, h = w = 61, one batched
    launch (the bench's), 3 pages x ~150k sampled pixels vs the oracle."""
    host, x = config3
    cnt = torch.zeros(2, dtype=torch.int64, device=DEV)
    m = ab.binarize_batched(method, x, 61, 61, k, 128.0, counters=cnt)
    torch.cuda.synchronize()
    for p in (0, 31, 63):
        rows, cols = sample_points(7016, 4960, 100_000, seed=p)
        ref = oracle.binarize_points(method, host[p], 61, 61, k, 128.0, -1, rows, cols)
        got = m[p].cpu().numpy()[rows, cols]
        assert np.array_equal(got, ref["mask"]), (method, p, int((got != ref["mask"]).sum()))
    assert int(cnt[0]) == 0  # no near ties on these pages (BASELINE.json: "zero expected")
    # any-size property: foreground is a minority (strokes ~10%) and not empty
    fg = 1.0 - m.float().mean().item()
    assert 0.02 < fg < 0.5


def test_config4_gigapixel_sampled_and_bands():
    """Config 4: 32768 x 32768, Sauvola k = 0.34, h = w = 101, forced uint64
    square sums, bit mask -- the whole image (N = 1 bench launch) vs the
    oracle at sampled pixels, and the 8-band decomposition (the N = 8 launch
    configuration, halos filled locally) bit-identical to the whole image."""
    H = W = 32768
    host = synth.page(H, W, synth.config_seed(4))
    buf = torch.zeros((H, W), dtype=torch.uint8, device=DEV)
    buf.copy_(torch.from_numpy(host))
    cnt = torch.zeros(2, dtype=torch.int64, device=DEV)
    whole = ab.sauvola(buf, 101, 101, 0.34, 128.0, packed=True, flags=abin.FORCE_U64_SQ, counters=cnt)
    torch.cuda.synchronize()
    rows, cols = sample_points(H, W, 150_000, seed=4, seam=432)
    # band seams of the 8-rank decomposition
    br = np.concatenate([np.arange(b - 3, b + 3) for b in range(4096, H, 4096)])
    rows = np.concatenate([rows, np.repeat(br, 64)])
    cols = np.concatenate([cols, np.random.default_rng(9).integers(0, W, br.size * 64)])
    ref = oracle.binarize_points("sauvola", host, 101, 101, 0.34, 128.0, -1, rows, cols)
    wb = whole.cpu().numpy()
    got = unpack(wb, W)[rows, cols]
    assert np.array_equal(got, ref["mask"]), int((got != ref["mask"]).sum())
    assert int(cnt[0]) == 0
    del buf
    parts = []
    for g in range(8):
        band = adist.make_band(H, W, 101, g, 8, device=DEV)
        band.buf.copy_(torch.from_numpy(host[band.r0 - band.top:band.r1 + band.bot]).to(DEV))
        parts.append(adist.run_band("sauvola", band, 101, 101, 0.34, 128.0, packed=True, rank=g, world=8,
                                    exchange=False, flags=abin.FORCE_U64_SQ).cpu().numpy())
        del band
    assert np.array_equal(np.concatenate(parts), wb)


@pytest.mark.parametrize("hw", [15, 31, 63, 127, 255])
def test_config2_window_sweep(hw):
    """Config 2: 3300 x 2550 letter page, the whole window sweep; the full
    page vs the oracle for the small windows, sampled pixels for the rest."""
    H, W = 3300, 2550
    host, x = device_pages(1, H, W, 2, False)
    m = ab.sauvola(x[0], hw, hw, 0.5, 128.0).cpu().numpy()
    if hw <= 31:
        assert np.array_equal(m, oracle.binarize("sauvola", host[0], hw, hw, 0.5, 128.0))
    else:
        rows, cols = sample_points(H, W, 60_000 if hw < 255 else 20_000, seed=hw)
        ref = oracle.binarize_points("sauvola", host[0], hw, hw, 0.5, 128.0, -1, rows, cols)
        assert np.array_equal(m[rows, cols], ref["mask"])


@pytest.mark.parametrize("q", [0.5, 0.1, 0.9])
def test_config5_quantile_sampled(q):
    """Config 5: 4096 x 4096, local median / P10 / P90 over 51 x 51, and the
    32-page batch (config 5b's launch) -- sampled pixels vs the sort-based
    oracle."""
    H = W = 4096
    P = 32 if q == 0.5 else 1
    host, x = device_pages(P, H, W, 5, False)
    m = ab.binarize_batched("quantile", x, 51, 51, q).cpu().numpy()
    for p in sorted({0, P - 1}):
        rows, cols = sample_points(H, W, 30_000, seed=int(q * 10) + p, seam=128)
        mref, _ = oracle.quantile_points(host[p], 51, 51, q, rows, cols)
        assert np.array_equal(m[p][rows, cols], mref), (q, p)


def test_bernsen_fullsize_sampled():
    """Bernsen (NEXT #1) on a config-5-sized page (4096 x 4096, 51 x 51) and a
    16-page batch, sampled pixels vs the direct extrema oracle."""
    H = W = 4096
    host, x = device_pages(16, H, W, 5, True)
    for contrast in (-1, 20):
        m = ab.binarize_batched("bernsen", x, 51, 51, float(contrast)).cpu().numpy()
        for p in (0, 15):
            rows, cols = sample_points(H, W, 30_000, seed=p + contrast + 2, seam=128)
            ref = oracle.bernsen_points(host[p], 51, 51, contrast, rows, cols)
            assert np.array_equal(m[p][rows, cols], ref), (contrast, p)
