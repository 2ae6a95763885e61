"""Khurshid and Phansalkar on the v5 kernel (-m gpu).

Table 1 rows PAPER.md:156-157.  With h <= 129, w <= 127 and (Phansalkar)
q >= 0 these rules run on the production v5 kernel: an fp32 residual from the
exact integer window sums, a certified bound derived per parameter set
(abin_api.cu filter_consts_v5; the bound itself is checked on 1.5e7 tuples
per set in test_gpu_filter_bound.py) and the IEEE-double Table-1 row for the
pixels inside it (fixup.cuh).  The mask must be the v3 kernel's (every pixel
in double, the same device routines) bit for bit, and the oracle's (Khurshid
uses only IEEE-exact operations: bit-exact; Phansalkar's exp may differ from
glibc's in the last ulp: mismatches only on near ties, R18).
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
SETS = {"khurshid": [(-0.1, 0), (0.2, 1), (-0.3, 1)],
        "phansalkar": [(0.25, 128.0, 3.0, 10.0 / 255.0), (-0.3, 64.0, -2.0, 0.5), (0.5, 128.0, 1.0, 0.0)]}


def to_dev(I):
    H, W = I.shape
    pitch = (W + 15) // 16 * 16
    buf = torch.zeros((H, pitch), dtype=torch.uint8, device=DEV)
    buf[:, :W] = torch.from_numpy(np.ascontiguousarray(I)).to(DEV)
    return buf[:, :W]


def check(rule, prm, I, h, w, packed=False):
    x = to_dev(I)
    c5 = torch.zeros(3, dtype=torch.int64, device=DEV)
    c3 = torch.zeros(3, dtype=torch.int64, device=DEV)
    got = ab.binarize_rule(rule, x, h, w, prm, packed=packed, counters=c5).cpu().numpy()
    v3 = ab.binarize_rule(rule, x, h, w, prm, packed=packed, counters=c3, flags=abin.V3_INTERNAL).cpu().numpy()
    bad = np.argwhere(got != v3)
    assert bad.size == 0, f"{rule}{prm} {I.shape} {h}x{w}: {len(bad)} v5/v3 mismatches, first {bad[:5].tolist()}"
    assert int(c5[0]) == int(c3[0])   # near ties (|I - t| < 1e-9): all reach the exact stage
    ref, t = oracle.binarize_rule(rule, I, h, w, prm, with_t=True)
    mask = np.unpackbits(got, axis=1)[:, :I.shape[1]] if packed else got   # MSB-first rows
    if rule == "khurshid":
        assert np.array_equal(mask, ref), (rule, prm, h, w, int((mask != ref).sum()))
    else:
        tie = np.abs(I.astype(np.float64) - t) < 1e-9
        assert not ((mask != ref) & ~tie).any(), (rule, prm, h, w)
    return c5.cpu().numpy()


@pytest.mark.parametrize("rule", sorted(SETS))
@pytest.mark.parametrize("w", [1, 2, 7, 16, 17, 31, 32, 33, 61, 64, 101, 127])
def test_rules_every_phase(rule, w):
    I = synth.page(70, 1000, synth.config_seed(7, w), stain=True)
    for prm in SETS[rule]:
        check(rule, prm, I, 15 if w > 3 else 3, w)


@pytest.mark.parametrize("h", [1, 2, 30, 64, 129])
def test_rules_window_heights(h):
    I = synth.page(150, 700, synth.config_seed(8, h), stain=True)
    check("khurshid", (-0.1, 0), I, h, 61)
    check("phansalkar", SETS["phansalkar"][0], I, h, 45)


def test_rules_packed_and_degenerate_pages():
    I = synth.page(64, 1333, synth.config_seed(9, 1))
    check("khurshid", (0.2, 1), I, 11, 61, packed=True)
    check("phansalkar", SETS["phansalkar"][0], I, 11, 61, packed=True)
    for g in (0, 255):
        C = np.full((64, 600), g, np.uint8)
        check("khurshid", (-0.1, 0), C, 5, 9)
        check("phansalkar", SETS["phansalkar"][1], C, 5, 9)
        C[::7, ::5] = 255 - g
        check("khurshid", (0.3, 1), C, 129, 127)
        check("phansalkar", SETS["phansalkar"][2], C, 129, 127)


def test_rules_near_ties_reach_the_exact_stage():
    # Khurshid with k = 0 is t = m: a constant page ties everywhere
    C = np.full((40, 500), 91, np.uint8)
    cnt = check("khurshid", (0.0, 0), C, 7, 7)
    assert cnt[0] == C.size
    # low contrast: thresholds close to the pixels
    rng = np.random.default_rng(3)
    I = (128 + rng.integers(-2, 3, size=(120, 800))).astype(np.uint8)
    check("khurshid", (-0.05, 1), I, 7, 7)
    check("phansalkar", (0.0, 128.0, 0.0, 0.0), I, 7, 7)   # t = m


def test_rules_outside_v5_stay_exact():
    # q < 0 (unbounded e^(-q m)) and wide windows: the per-pixel double path
    I = synth.page(60, 500, synth.config_seed(9, 2), stain=True)
    check("phansalkar", (0.25, 128.0, 3.0, -0.01), I, 9, 9)
    check("khurshid", (-0.1, 0), I, 9, 201)


# ---- Rais (the bound formed per page from M S) and Feng (gamma >= 1) on v5 behind their
# certified filters: the same masks as the v3 kernel's per-pixel double
EXACT_SETS = {"feng": [(0.12, 0.015, 0.01, 2.0, 128.0), (0.2, 0.05, 0.02, 1.5, 64.0), (0.12, 0.015, 0.01, 0.5, 128.0)],
              "rais": [()]}


@pytest.mark.parametrize("rule", sorted(EXACT_SETS))
def test_feng_rais_on_v5(rule):
    """Masks and near-tie counts equal the v3 kernel's (every pixel in double)
    and the oracle's (Rais: IEEE-exact operations, bit-exact; Feng's pow may
    differ from glibc's in the last ulp: near ties excluded, R18),
    over the strip geometry classes, borders and random pages."""
    rng = np.random.default_rng(31)
    for prm in EXACT_SETS[rule]:
        for (H, W), (h, w) in [((130, 333), (15, 15)), ((200, 517), (61, 61)), ((77, 450), (40, 33)),
                               ((150, 600), (129, 127)), ((40, 70), (9, 100)), ((96, 512), (4, 32))]:
            I = synth.page(H, W, synth.config_seed(10, H + W), stain=True)
            x = to_dev(I)
            for packed in (False, True):
                c5 = torch.zeros(2, dtype=torch.int64, device=DEV)
                c3 = torch.zeros(2, dtype=torch.int64, device=DEV)
                got = ab.binarize_rule(rule, x, h, w, prm, packed=packed, counters=c5).cpu().numpy()
                v3 = ab.binarize_rule(rule, x, h, w, prm, packed=packed, counters=c3,
                                      flags=abin.V3_INTERNAL).cpu().numpy()
                assert np.array_equal(got, v3), (rule, prm, H, W, h, w, packed)
                assert int(c5[0]) == int(c3[0])
            ref, t = oracle.binarize_rule(rule, I, h, w, prm, with_t=True)
            if rule == "rais":
                assert np.array_equal(got if not packed else ab.binarize_rule(rule, x, h, w, prm).cpu().numpy(), ref)
            else:
                g = ab.binarize_rule(rule, x, h, w, prm).cpu().numpy()
                tie = np.abs(I.astype(np.float64) - t) < 1e-9
                assert not ((g != ref) & ~tie).any(), (rule, prm, h, w)
        # random pixels (no structure): the rules' fractions and powers over the whole range
        R = rng.integers(0, 256, size=(90, 300), dtype=np.uint8)
        x = to_dev(R)
        got = ab.binarize_rule(rule, x, 21, 37, prm).cpu().numpy()
        v3 = ab.binarize_rule(rule, x, 21, 37, prm, flags=abin.V3_INTERNAL).cpu().numpy()
        assert np.array_equal(got, v3), (rule, prm)
