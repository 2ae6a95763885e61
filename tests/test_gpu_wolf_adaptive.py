"""Wolf with the image-adaptive R (NEXT #3, R21) on the GPU (-m gpu):
abin_max_s equals the oracle's max s bit for bit (the canonical double s of
the maximising pixel), and abin_wolf_adaptive's mask equals the oracle's
Wolf mask with that R -- on document pages, random pages, constant pages
(R = +inf), maximum-variance pages and band decompositions."""
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


def to_dev(I):
    H, W = I.shape
    buf = torch.zeros((H, (W + 15) // 16 * 16), dtype=torch.uint8, device=DEV)
    buf[:, :W] = torch.from_numpy(np.ascontiguousarray(I)).to(DEV)
    return buf[:, :W]


def pages():
    yield "doc", synth.page(300, 700, synth.config_seed(3, 81), stain=True), (31, 31)
    yield "doc61", synth.page(400, 1100, synth.config_seed(3, 82), stain=True), (61, 61)
    yield "random", synth.uniform_random(120, 333, 83), (15, 9)
    yield "constant", synth.constant(90, 200, 77), (11, 11)
    J = np.zeros((64, 256), np.uint8)
    J[:, ::2] = 255                                   # every 2x2 window: s = 127.5
    yield "max_variance", J, (2, 2)
    yield "even", synth.page(150, 500, synth.config_seed(3, 84)), (32, 20)


@pytest.mark.parametrize("name,I,hw", list(pages()))
def test_max_s_and_wolf_adaptive(name, I, hw):
    h, w = hw
    x = to_dev(I)
    ms = ab.max_s(x, h, w)
    assert ms == oracle.max_s(I, h, w), (name, ms, oracle.max_s(I, h, w))   # bit-exact double
    mask, R = ab.wolf_adaptive(x, h, w, 0.5)
    R_ref = oracle.adaptive_R(I, h, w)
    assert R == R_ref
    want = oracle.binarize("wolf", I, h, w, 0.5, R_ref)
    assert np.array_equal(mask.cpu().numpy(), want), name
    if name == "constant":
        assert R == float("inf") and (mask.cpu().numpy() == 0).all()


def test_max_s_over_bands():
    I = synth.page(500, 600, synth.config_seed(3, 85), stain=True)
    h, w = 41, 33
    o, u = (h + 1) // 2, h // 2
    whole = oracle.max_s(I, h, w)
    got = []
    for r0, r1 in [(0, 140), (140, 333), (333, 500)]:
        top, bot = min(o - 1, r0), min(u, 500 - r1)
        held = to_dev(np.ascontiguousarray(I[r0 - top:r1 + bot]))
        got.append(ab.max_s(held, h, w, row0=r0, H_global=500, halo_top=top, halo_bot=bot))
    assert max(got) == whole


def test_max_s_validation():
    # (effective windows: clamped to the image, so the image must be larger)
    x = torch.zeros((400, 512), dtype=torch.uint8, device=DEV)
    with pytest.raises(abin.AbinError):
        ab.max_s(x, 131, 9)          # h beyond the v5 domain
    with pytest.raises(abin.AbinError):
        ab.max_s(x, 9, 129)          # w beyond the v5 domain
    assert ab.max_s(x[:40], 131, 9) == 0.0   # clamped to 40 + 40 rows: inside the domain
