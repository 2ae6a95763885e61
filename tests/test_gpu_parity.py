"""GPU parity (-m gpu): the CUDA path (through the C ABI) against the CPU
oracle, element by element on seeded inputs.

Bars (BASELINE.json north_star): masks, window sums, counts and quantiles
bit-exact; thresholds (fp64, identical expression order, no contraction)
within 1e-12 relative -- in practice bit-identical, which is also checked;
near-ties (|I - t| < 1e-9) counted.
"""
import functools
import zlib

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
T_RTOL = 1e-12


def to_dev(I: np.ndarray, pitch: int = None) -> torch.Tensor:
    """Copy a (H, W) page to the device; pitch=None: 16-byte padded pitch
    (TMA path), pitch=W: tight rows (generic loader when W % 16 != 0)."""
    H, W = I.shape
    if pitch is None:
        pitch = (W + 15) // 16 * 16
    buf = torch.zeros((H, pitch), dtype=torch.uint8, device=DEV)
    buf[:, :W] = torch.from_numpy(np.ascontiguousarray(I)).to(DEV)
    return buf[:, :W]


PARAMS = {"sauvola": (0.5, 128.0), "niblack": (-0.2, 128.0), "wolf": (0.5, 128.0)}


def run(method, x, h, w, packed=False, flags=0, counters=None):
    k, R = PARAMS[method]
    if method == "sauvola":
        return ab.sauvola(x, h, w, k, R, packed=packed, flags=flags, counters=counters)
    if method == "niblack":
        return ab.niblack(x, h, w, k, packed=packed, flags=flags, counters=counters)
    return ab.wolf(x, h, w, k, R, packed=packed, flags=flags, counters=counters)


def check_full(method, I, h, w, pitch=None, packed=False, stats=True):
    k, R = PARAMS[method]
    ref = oracle.binarize(method, I, h, w, k, R, stats=stats)
    x = to_dev(I, pitch)
    cnt = torch.zeros(2, dtype=torch.int64, device=DEV)
    m = run(method, x, h, w, packed=packed, counters=cnt)
    got = m.cpu().numpy()
    want = ref["mask"] if stats else ref
    if packed:
        want = oracle.pack_bits(want)
    assert np.array_equal(got, want), f"{method} mask mismatch {I.shape} h={h} w={w} packed={packed}: " \
                                      f"{int((got != want).sum())} px"
    if stats:
        assert int(cnt[0]) == ref["near_tie"]
        s = ab.stats(method, x, h, w, k, R)
        assert np.array_equal(s["c"].cpu().numpy().astype(np.uint64), ref["c"])
        assert np.array_equal(s["d"].cpu().numpy().astype(np.uint64), ref["d"])
        assert np.array_equal(s["n"].cpu().numpy().astype(np.uint64), ref["n"])
        t = s["t"].cpu().numpy()
        rel = np.abs(t - ref["t"]) / np.maximum(np.abs(ref["t"]), 1e-300)
        assert rel.max() <= T_RTOL
        assert np.array_equal(t, ref["t"]), "thresholds are not bit-identical"
        assert np.array_equal(s["mask"].cpu().numpy(), ref["mask"])


# ------------------------------------------------------------------ config 1

@pytest.mark.parametrize("packed", [False, True])
def test_config1_full_page(packed):
    I = synth.page(512, 512, synth.config_seed(1))
    check_full("sauvola", I, 32, 32, packed=packed)


# ------------------------------------------------------------------ SPEC grid

SPEC_WINDOWS = [(1, 1), (2, 2), (3, 3), (2, 5), (5, 2), (31, 31), (64, 64), (100, 7)]
SPEC_SHAPES = [(1, 1), (7, 9), (33, 20), (3, 200), (200, 3), (64, 64)]


@pytest.mark.parametrize("method", ["sauvola", "niblack", "wolf"])
@pytest.mark.parametrize("hw", SPEC_WINDOWS)
def test_spec_grid(method, hw):
    rng = np.random.default_rng(zlib.crc32(f"{method}{hw}".encode()))
    for (H, W) in SPEC_SHAPES:
        I = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
        for pitch in (None, W):
            check_full(method, I, hw[0], hw[1], pitch=pitch, stats=(pitch is None))


@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("shape,hw", [((300, 2100), (61, 61)), ((1030, 333), (32, 17)), ((77, 1500), (101, 101)),
                                      ((260, 900), (255, 255)), ((129, 3000), (15, 400))])
def test_multi_tile_ragged(shape, hw, packed):
    # several strips and row bands, ragged right/bottom tails, odd widths
    I = synth.page(*shape, seed=synth.config_seed(7, shape[0]), stain=True)
    for method in ("sauvola", "niblack"):
        check_full(method, I, *hw, packed=packed, stats=not packed)


def test_generic_loader_equals_tma_path():
    I = synth.page(200, 1000, synth.config_seed(8))
    a = run("sauvola", to_dev(I), 31, 31).cpu().numpy()
    b = run("sauvola", to_dev(I, pitch=1000), 31, 31).cpu().numpy()     # 1000 % 16 != 0
    buf = torch.zeros(200 * 1000 + 1, dtype=torch.uint8, device=DEV)    # misaligned base
    xm = buf[1:].view(200, 1000)
    xm.copy_(torch.from_numpy(I).to(DEV))
    c = run("sauvola", xm, 31, 31).cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(a, c)
    # unaligned rows are re-pitched for TMA; NO_TMA_INTERNAL keeps the generic loader
    for x in (to_dev(I, pitch=1000), xm, to_dev(I)):
        for method in ("sauvola", "niblack", "wolf"):
            g = run(method, x, 31, 31, flags=abin.NO_TMA_INTERNAL).cpu().numpy()
            assert np.array_equal(g, run(method, to_dev(I), 31, 31).cpu().numpy()), method
    # unaligned page batches (page stride 1000 * 200 + 3) through the re-pitch path
    pb = torch.zeros(3 * (200 * 1000 + 3), dtype=torch.uint8, device=DEV)
    pages = torch.as_strided(pb, (3, 200, 1000), (200 * 1000 + 3, 1000, 1))
    pages.copy_(torch.from_numpy(np.stack([I, I[::-1].copy(), 255 - I])).to(DEV))
    mb = ab.binarize_batched("sauvola", pages, 31, 31, 0.5, 128.0).cpu().numpy()
    for k, P in enumerate([I, I[::-1].copy(), 255 - I]):
        assert np.array_equal(mb[k], oracle.binarize("sauvola", P, 31, 31, 0.5, 128.0)), k


# ------------------------------------------------------------------ adversarial

def test_low_contrast_niblack():
    # 128 +- 2: Niblack thresholds land within ~1e-13 of pixel values
    I = synth.low_contrast(97, 131, 5)
    for hw in [(3, 3), (7, 5), (31, 31)]:
        check_full("niblack", I, *hw)


@pytest.mark.parametrize("g", [0, 1, 128, 255])
def test_constant_images(g):
    I = synth.constant(45, 70, g)
    for method in ("sauvola", "niblack", "wolf"):
        check_full(method, I, 9, 12)


def test_one_by_one_and_huge_windows():
    I = synth.uniform_random(50, 60, 6)
    for method in ("sauvola", "niblack", "wolf"):
        check_full(method, I, 1, 1)
        check_full(method, I, 99, 119)        # whole-image window from every pixel
        check_full(method, I, 500, 3)         # taller than the image


def test_accumulator_bounds_all_255():
    # h = w = 257 on an all-255 image
    I = synth.constant(300, 300, 255)
    check_full("sauvola", I, 257, 257)


def test_even_and_odd_windows_asymmetry():
    I = synth.page(120, 150, 17)
    for hw in [(4, 4), (4, 5), (5, 4), (6, 9), (32, 32), (33, 33)]:
        check_full("sauvola", I, *hw)


# ------------------------------------------------------------------ stats / misc

def test_wolf_global_min_on_device():
    P = synth.pages(3, 64, 80, synth.config_seed(3), stain=True)
    x = torch.from_numpy(P).to(DEV)
    L = ab.global_min(x).cpu().numpy()
    assert list(L) == [int(p.min()) for p in P]


def test_forced_u64_square_sums_equal_u32():
    I = synth.page(300, 400, 23)
    x = to_dev(I)
    a = ab.sauvola(x, 101, 101, 0.34, 128.0, packed=True).cpu().numpy()
    b = ab.sauvola(x, 101, 101, 0.34, 128.0, packed=True, flags=abin.FORCE_U64_SQ).cpu().numpy()
    assert np.array_equal(a, b)
    assert np.array_equal(a, oracle.pack_bits(oracle.binarize("sauvola", I, 101, 101, 0.34, 128.0)))


def test_batched_pages_equal_single_pages():
    P = synth.pages(5, 130, 210, synth.config_seed(3), stain=True)
    x = torch.from_numpy(P).to(DEV)
    for method, (k, R) in PARAMS.items():
        mb = ab.binarize_batched(method, x, 61, 61, k, R).cpu().numpy()
        for p in range(5):
            ref = oracle.binarize(method, P[p], 61, 61, k, R)
            assert np.array_equal(mb[p], ref), (method, p)


def test_band_decomposition_equals_whole_image():
    # K7: G row bands with halo rows (o-1 above, u below) reproduce the
    # whole-image mask bit for bit (single process, one GPU).
    I = synth.page(1000, 700, 29)
    Hg = I.shape[0]
    for (h, w), method in [((101, 101), "sauvola"), ((32, 32), "niblack"), ((51, 51), "quantile")]:
        k, R = PARAMS.get(method, (0.5, 128.0))
        o, u = (h + 1) // 2, h // 2
        if method == "quantile":
            whole, _ = oracle.quantile(I, h, w, 0.5)
        else:
            whole = oracle.binarize(method, I, h, w, k, R)
        for G in (2, 3, 8):
            bounds = np.linspace(0, Hg, G + 1).astype(int)
            parts = []
            for g in range(G):
                r0, r1 = bounds[g], bounds[g + 1]
                top = min(o - 1, r0)
                bot = min(u, Hg - r1)
                held = to_dev(np.ascontiguousarray(I[r0 - top:r1 + bot]))
                m = ab.binarize_band(method, held, r0, Hg, top, bot, h, w, 0.5 if method == "quantile" else k, R)
                parts.append(m.cpu().numpy())
            assert np.array_equal(np.concatenate(parts), whole), (method, G)


# ------------------------------------------------------------------ quantile

@pytest.mark.parametrize("q", [0.5, 0.1, 0.9, 1.0, 0.001])
def test_quantile_small(q):
    rng = np.random.default_rng(int(q * 1000))
    for (H, W), (h, w) in [((33, 41), (5, 5)), ((64, 200), (51, 51)), ((7, 300), (4, 9)), ((100, 3), (3, 100))]:
        I = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
        mref, Qref = oracle.quantile(I, h, w, q)
        for pitch in (None, W):
            x = to_dev(I, pitch)
            m = ab.quantile(x, h, w, q).cpu().numpy()
            assert np.array_equal(m, mref)
            mb = ab.quantile(x, h, w, q, packed=True).cpu().numpy()
            assert np.array_equal(mb, oracle.pack_bits(mref))
        s = ab.stats("quantile", to_dev(I), h, w, q)
        assert np.array_equal(s["t"].cpu().numpy(), Qref.astype(np.float64))


@pytest.mark.parametrize("kernel", ["v5", "pair", "single"])
@pytest.mark.parametrize("hw", [(3, 3), (12, 7), (51, 51), (125, 40), (126, 40), (30, 128), (30, 129)])
def test_quantile_all_kernels(monkeypatch, kernel, hw):
    """The v5 kernel (quantile5.cuh, default for masks with h <= 255,
    w <= 127), the paired-column kernel (k_quantile2: forced with the
    Q2_INTERNAL hook where its packing allows, h <= 125, w <= 128) and the
    single-column kernel (ABIN_QUANTILE_SINGLE, and beyond those limits)
    against the oracle: odd widths (a last thread with one active column), bit
    masks, a page batch and the Q statistics; windows on both sides of the
    limits."""
    flags = 0 if kernel == "v5" else abin.Q2_INTERNAL
    if kernel == "single":
        monkeypatch.setenv("ABIN_QUANTILE_SINGLE", "1")
    h, w = hw
    pages = _quantile_pages()
    buf = torch.zeros((2, 120, 272), dtype=torch.uint8, device=DEV)  # 16-byte aligned rows (v5)
    buf[:, :, :261] = torch.from_numpy(pages).to(DEV)
    x = buf[:, :, :261]
    for q in (0.5, 0.1):
        mb = ab.binarize_batched("quantile", x, h, w, q, flags=flags).cpu().numpy()
        bits = ab.binarize_batched("quantile", x, h, w, q, packed=True, flags=flags).cpu().numpy()
        for p in range(2):
            mref, Qref = _quantile_ref(p, h, w, q)
            assert np.array_equal(mb[p], mref), (hw, q, p)
            assert np.array_equal(bits[p], oracle.pack_bits(mref)), (hw, q, p)
        s = ab.stats("quantile", to_dev(pages[1]), h, w, q)
        assert np.array_equal(s["t"].cpu().numpy(), Qref.astype(np.float64))


@functools.lru_cache(maxsize=None)
def _quantile_pages():
    rng = np.random.default_rng(5)
    pages = np.stack([synth.page(120, 261, synth.config_seed(5) + k) for k in range(2)])
    pages[1, 40:90, 100:200] = rng.integers(0, 256, size=(50, 100), dtype=np.uint8)
    return pages


@functools.lru_cache(maxsize=None)
def _quantile_ref(p, h, w, q):
    return oracle.quantile(_quantile_pages()[p], h, w, q)


def test_quantile_document_page():
    I = synth.page(300, 500, synth.config_seed(5))
    for q in (0.5, 0.1, 0.9):
        mref, _ = oracle.quantile(I, 51, 51, q)
        m = ab.quantile(to_dev(I), 51, 51, q).cpu().numpy()
        assert np.array_equal(m, mref), q


# ------------------------------------------------------------ multi-GPU driver

@pytest.mark.parametrize("G,h,w,packed", [(4, 101, 101, True), (3, 32, 31, False), (2, 9, 8, False)])
def test_driver_bands_emulated_on_one_gpu(G, h, w, packed):
    """paper_1905_13038_b200.dist.run_band on G emulated ranks (halos filled
    from the global image instead of NCCL): interior / top / bottom strips
    launched as on the real multi-GPU path; the concatenated masks equal the
    oracle's whole-image mask."""
    from paper_1905_13038_b200 import dist as adist
    H, W = 403, 700
    I = synth.page(H, W, synth.config_seed(4, 3))
    k = 0.34
    parts = []
    for g in range(G):
        band = adist.make_band(H, W, h, g, G, device=DEV)
        band.buf.copy_(torch.from_numpy(I[band.r0 - band.top:band.r1 + band.bot]).to(DEV))
        parts.append(adist.run_band("sauvola", band, h, w, k, 128.0, packed=packed, rank=g, world=G,
                                    exchange=False, flags=abin.FORCE_U64_SQ).cpu().numpy())
    got = np.concatenate(parts, axis=0)
    want = oracle.binarize("sauvola", I, h, w, k, 128.0)
    if packed:
        want = oracle.pack_bits(want)
    assert np.array_equal(got, want)


# ------------------------------------------------------------ host buffers

@pytest.mark.parametrize("packed,pad", [(False, 0), (True, 0), (False, 5)])
def test_host_io_batched_equals_device_path(packed, pad):
    """ABIN_HOST_IO: pinned host pages in, host masks out, streamed through
    device staging -- identical to the device-resident call (and the oracle)."""
    P, H, W = 7, 230, 333
    pages = synth.pages(P, H, W, synth.config_seed(3), stain=True)
    hbuf = torch.zeros((P, H, W + pad), dtype=torch.uint8).pin_memory()
    hbuf[:, :, :W] = torch.from_numpy(pages)
    hin = hbuf[:, :, :W]
    cols = (W + 7) // 8 if packed else W
    hout = torch.zeros((P, H, cols + pad), dtype=torch.uint8).pin_memory()
    fmt = abin.MASK_BITS if packed else abin.MASK_U8
    rc = abin.raw().abin_binarize_batched(
        abin.SAUVOLA, abin.ctypes.c_void_p(hin.data_ptr()), hin.stride(0), abin.ctypes.c_void_p(hout.data_ptr()),
        hout.stride(0), P, H, W, hin.stride(1), hout.stride(1), fmt, 31, 31, 0.5, 128.0, -1, abin.HOST_IO, None,
        abin.ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    got = hout[:, :, :cols].numpy()
    for p in range(P):
        want = oracle.binarize("sauvola", pages[p], 31, 31, 0.5, 128.0)
        assert np.array_equal(got[p], oracle.pack_bits(want) if packed else want), p


@pytest.mark.parametrize("method,p0,p1,L", [("sauvola", 0.5, 128.0, -1), ("niblack", -0.2, 0.0, -1),
                                             ("wolf", 0.5, 128.0, 7), ("quantile", 0.5, 0.0, -1),
                                             ("bernsen", 15.0, 0.0, -1)])
@pytest.mark.parametrize("packed,pad", [(False, 0), (True, 3)])
def test_host_io_row_bands(monkeypatch, method, p0, p1, L, packed, pad):
    """ABIN_HOST_IO with pages larger than a chunk: each page travels as row
    bands with their window halos (here ~20 KB chunks: 5 bands per page), and
    the masks equal the device-resident call's."""
    monkeypatch.setenv("ABIN_HOSTIO_CHUNK_BYTES", "20000")
    P, H, W = 3, 230, 333
    pages = synth.pages(P, H, W, synth.config_seed(3), stain=True)
    pages[1, 100:140] = 200                                   # flat rows: Niblack ties, fixup queue
    hbuf = torch.zeros((P, H, W + pad), dtype=torch.uint8).pin_memory()
    hbuf[:, :, :W] = torch.from_numpy(pages)
    hin = hbuf[:, :, :W]
    cols = (W + 7) // 8 if packed else W
    hout = torch.zeros((P, H, cols + pad), dtype=torch.uint8).pin_memory()
    fmt = abin.MASK_BITS if packed else abin.MASK_U8
    rc = abin.raw().abin_binarize_batched(
        abin.METHODS[method], abin.ctypes.c_void_p(hin.data_ptr()), hin.stride(0),
        abin.ctypes.c_void_p(hout.data_ptr()), hout.stride(0), P, H, W, hin.stride(1), hout.stride(1), fmt, 31, 25,
        p0, p1, L, abin.HOST_IO, None, abin.ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    monkeypatch.delenv("ABIN_HOSTIO_CHUNK_BYTES")
    dev = torch.from_numpy(pages).to(DEV)
    if method == "wolf":
        want = ab.binarize_batched(method, dev, 31, 25, p0, p1, L=L, packed=packed)
    else:
        want = ab.binarize_batched(method, dev, 31, 25, p0, p1, packed=packed)
    assert np.array_equal(hout[:, :, :cols].numpy(), want.cpu().numpy())
    if method == "sauvola":
        for p in range(P):
            ref = oracle.binarize("sauvola", pages[p], 31, 25, 0.5, 128.0)
            assert np.array_equal(want[p].cpu().numpy(), oracle.pack_bits(ref) if packed else ref)


# ------------------------------------------------------------ Bernsen (NEXT #1)

@pytest.mark.parametrize("contrast", [-1, 15])
@pytest.mark.parametrize("single", [False, True])
def test_bernsen_small(monkeypatch, contrast, single):
    """Bernsen midrange: the window-independent row/column
    kernels (default) and the histogram kernels (Q2_INTERNAL: the paired
    k_quantile2, k_quantile with ABIN_QUANTILE_SINGLE) vs the direct extrema
    oracle: random and document images, odd/even windows, windows larger than
    the image, byte and bit masks, tight and padded pitches."""
    if single:
        monkeypatch.setenv("ABIN_QUANTILE_SINGLE", "1")
    rng = np.random.default_rng(contrast + 2)
    cases = [((33, 41), (5, 5)), ((64, 200), (51, 51)), ((7, 300), (4, 9)), ((100, 3), (3, 100)),
             ((130, 257), (16, 31))]
    for (H, W), (h, w) in cases:
        for I in (rng.integers(0, 256, size=(H, W), dtype=np.uint8),
                  synth.page(H, W, synth.config_seed(6, H), stain=True)):
            ref, lo, hi = oracle.bernsen(I, h, w, contrast)
            for pitch in (None, W):
                x = to_dev(I, pitch)
                for fl in (0, abin.Q2_INTERNAL):
                    assert np.array_equal(ab.bernsen(x, h, w, contrast, flags=fl).cpu().numpy(), ref)
                    assert np.array_equal(ab.bernsen(x, h, w, contrast, packed=True, flags=fl).cpu().numpy(),
                                          oracle.pack_bits(ref))
            s = ab.stats("bernsen", to_dev(I), h, w, float(contrast))
            assert np.array_equal(s["t"].cpu().numpy(), 0.5 * (lo.astype(np.float64) + hi))
            assert np.array_equal(s["mask"].cpu().numpy(), ref)


def test_bernsen_constant_and_bands():
    I = synth.constant(50, 70, 91)
    assert (ab.bernsen(to_dev(I), 9, 9).cpu().numpy() == 0).all()
    assert (ab.bernsen(to_dev(I), 9, 9, contrast=1).cpu().numpy() == 1).all()
    J = synth.page(600, 400, synth.config_seed(6, 1))
    whole, _, _ = oracle.bernsen(J, 21, 21, 20)
    for G in (2, 5):
        bounds = np.linspace(0, 600, G + 1).astype(int)
        parts = []
        for g in range(G):
            r0, r1 = bounds[g], bounds[g + 1]
            top, bot = min(10, r0), min(10, 600 - r1)
            held = to_dev(np.ascontiguousarray(J[r0 - top:r1 + bot]))
            parts.append(ab.binarize_band("bernsen", held, r0, 600, top, bot, 21, 21, 20.0).cpu().numpy())
        assert np.array_equal(np.concatenate(parts), whole)
    P = synth.pages(3, 90, 130, synth.config_seed(6, 2))
    mb = ab.binarize_batched("bernsen", torch.from_numpy(P).to(DEV), 15, 15, -1.0).cpu().numpy()
    for p in range(3):
        assert np.array_equal(mb[p], oracle.bernsen(P[p], 15, 15)[0])


# ------------------------------------------------ Table 1 rules (NEXT #2)

RULE_PARAMS = {"feng": (0.85, 0.2, 0.05, 2.0, 64.0), "rais": (), "khurshid": (-0.1, 0),
               "phansalkar": (0.25, 128.0, 3.0, 10.0 / 255.0)}


@pytest.mark.parametrize("rule", sorted(RULE_PARAMS))
def test_table1_rules(rule):
    """Feng / Rais / Khurshid / Phansalkar decided in IEEE
    double on the GPU vs the oracle.  Rais and Khurshid use only IEEE-exact
    operations: masks bit-exact.  Feng and Phansalkar call pow / exp (device
    <= 2 ulp vs glibc): masks bit-exact except pixels within 1e-9 of the
    oracle's threshold (R18)."""
    prm = RULE_PARAMS[rule]
    cases = [((300, 700), (61, 61), None), ((257, 333), (32, 17), 333), ((90, 1200), (15, 600), None),
             ((64, 64), (1, 1), None)]
    for (H, W), (h, w), pitch in cases:
        I = synth.page(H, W, synth.config_seed(3, H), stain=True)
        ref, t = oracle.binarize_rule(rule, I, h, w, prm, with_t=True)
        got = ab.binarize_rule(rule, to_dev(I, pitch), h, w, prm).cpu().numpy()
        tie = np.abs(I.astype(np.float64) - t) < 1e-9
        if rule in ("rais", "khurshid"):
            assert np.array_equal(got, ref), (rule, H, W, int((got != ref).sum()))
        else:  # any mismatch must sit on a near tie (pow / exp last-ulp differences)
            assert not ((got != ref) & ~tie).any(), (rule, H, W)
        gb = ab.binarize_rule(rule, to_dev(I, pitch), h, w, prm, packed=True).cpu().numpy()
        assert np.array_equal(gb, oracle.pack_bits(got))
    if rule == "khurshid":  # N = n variant
        I = synth.page(120, 200, synth.config_seed(3, 7))
        assert np.array_equal(ab.binarize_rule(rule, to_dev(I), 9, 9, (-0.1, 1)).cpu().numpy(),
                              oracle.binarize_rule(rule, I, 9, 9, (-0.1, 1)))


def test_table1_rules_validation():
    x = torch.zeros((8, 8), dtype=torch.uint8, device=DEV)
    with pytest.raises(abin.AbinError):
        ab.binarize_rule("feng", x, 3, 3, (0.5, 0.2, 0.05))          # too few params
    with pytest.raises(abin.AbinError):
        ab.binarize_rule("phansalkar", x, 3, 3, (0.25, 0.0, 3.0, 0.1))  # R <= 0


# ------------------------------------------------------------ Otsu (NEXT #4)

def test_otsu_equals_oracle():
    """Otsu's global threshold: the device histogram + the
    IEEE-double scan in the oracle's order give the same t and mask."""
    cases = [synth.page(300, 777, synth.config_seed(9, 1), stain=True), synth.uniform_random(129, 130, 4),
             synth.constant(40, 50, 33), synth.page(7016, 4960, synth.config_seed(3), stain=True)]
    for I in cases:
        t, ref = oracle.otsu(I)
        for pitch in (None, I.shape[1]):
            m, tt = ab.otsu(to_dev(I, pitch))
            assert int(tt.item()) == t
            assert np.array_equal(m.cpu().numpy(), ref)
        mb, _ = ab.otsu(to_dev(I), packed=True)
        assert np.array_equal(mb.cpu().numpy(), oracle.pack_bits(ref))


def test_wide_window_kernel():
    """Effective windows wider than 495 columns take the CTA-strip kernel
    (moments_wide.cuh): Sauvola / Niblack / Wolf against the oracle."""
    I = synth.page(150, 1400, synth.config_seed(7, 77), stain=True)
    for method in ("sauvola", "niblack", "wolf"):
        check_full(method, I, 33, 601, stats=False)
        check_full(method, I, 8, 1000, packed=True, stats=False)


@pytest.mark.parametrize("W", [704, 690])
@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("cap", [None, 1, 5000])
def test_fixup_queue_and_overflow(monkeypatch, packed, cap, W):
    """The v4 kernel queues the pixels its fp32 filter cannot decide; the
    fixup kernel decides them exactly.  On a near-constant page Niblack's
    threshold equals most pixel values (near ties everywhere), so the queue
    holds tens of thousands of pixels: cap=None is the production queue,
    cap=1 / 5000 force the overflow follow-up (the v3 kernel re-does the call
    exactly).  All three: masks bit-exact vs the oracle, near ties counted
    exactly once.  W = 690: 87-byte bit-mask rows, so the fixup's 32-bit
    atomics straddle rows."""
    if cap is not None:
        monkeypatch.setenv("ABIN_QUEUE_CAP", str(cap))
    rng = np.random.default_rng(17)
    P, H = 3, 300
    pages = np.full((P, H, W), 128, np.uint8)
    sel = rng.random((P, H, W)) < 2e-4
    pages[sel] = rng.integers(0, 256, int(sel.sum()), dtype=np.uint8)
    buf = torch.zeros((P, H, W), dtype=torch.uint8, device=DEV)
    buf.copy_(torch.from_numpy(pages))
    cnt = torch.zeros(2, dtype=torch.int64, device=DEV)
    m = ab.binarize_batched("niblack", buf, 31, 31, -0.2, 128.0, packed=packed, counters=cnt).cpu().numpy()
    near = 0
    for p in range(P):
        ref = oracle.binarize("niblack", pages[p], 31, 31, -0.2, 128.0, stats=True)
        want = oracle.pack_bits(ref["mask"]) if packed else ref["mask"]
        assert np.array_equal(m[p], want), (p, int((m[p] != want).sum()))
        near += ref["near_tie"]
    assert near > 10_000
    assert int(cnt[0]) == near


@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("bands", [False, True])
def test_host_io_touches_only_row_bytes(monkeypatch, packed, bands):
    """ABIN_HOST_IO with 16-aligned padded pitches (the linear-copy case):
    the input buffer ends right after the last row's W bytes, and the output
    rows' padding bytes and the bytes after the last row are not written
    (the copies once moved whole pitches)."""
    if bands:
        monkeypatch.setenv("ABIN_HOSTIO_CHUNK_BYTES", "20000")
    P, H, W = 3, 120, 400
    ip, op = 416, 432                                # 16-aligned pitches, padded
    cols = (W + 7) // 8 if packed else W
    pages = synth.pages(P, H, W, synth.config_seed(3, 77), stain=True)
    in_len = (P * H - 1) * ip + W                    # nothing after the last row
    out_len = (P * H - 1) * op + cols + 64           # 64 sentinel bytes after the last row
    hin = torch.full((in_len,), 0xCD, dtype=torch.uint8).pin_memory()
    hv = hin.numpy()
    for p in range(P):
        for i in range(H):
            o = (p * H + i) * ip
            hv[o:o + W] = pages[p, i]
    hout = torch.full((out_len,), 0xAB, dtype=torch.uint8).pin_memory()
    rc = abin.raw().abin_binarize_batched(
        abin.SAUVOLA, abin.ctypes.c_void_p(hin.data_ptr()), H * ip, abin.ctypes.c_void_p(hout.data_ptr()), H * op, P,
        H, W, ip, op, abin.MASK_BITS if packed else abin.MASK_U8, 31, 31, 0.5, 128.0, -1, abin.HOST_IO, None,
        abin.ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    ov = hout.numpy()
    for p in range(P):
        want = oracle.binarize("sauvola", pages[p], 31, 31, 0.5, 128.0)
        want = oracle.pack_bits(want) if packed else want
        for i in range(H):
            o = (p * H + i) * op
            assert np.array_equal(ov[o:o + cols], want[i]), (p, i)
            pad_end = min(o + op, out_len)
            assert (ov[o + cols:pad_end] == 0xAB).all(), (p, i)   # padding untouched
    assert (ov[(P * H - 1) * op + cols:] == 0xAB).all()
