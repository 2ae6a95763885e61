"""The certified fp32 filter's error bound, checked directly (-m gpu).

The v5 kernel decides a pixel in fp32 when its residual e~ = I - t~ is
farther from 0 than a host-derived bound, and queues it for the exact stages
otherwise.  Masks equal the fp64 decision only if the
bound holds: |e~ - e*| <= bound, e* = I - t(c, d, n) exactly.  Here the
production arithmetic (abin_probe_filter runs the kernel's own device
function on given tuples) is compared with e* evaluated on the host from the
exact integers (V = n d - c^2 in int64, then 80-bit long double), on 1.08e8
random realizable tuples (n = ncol nrow within the v5 domain, c in [0, 255 n],
d in [c^2/n, 255 c], I in [0, 255]) plus adversarial ones: near ties
(I = round(t*)), minimum-variance and constant windows, maximum-variance
windows, the smallest and largest counts.  SURVEY section 8(c) test (ii).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1905_13038_b200 import abin  # noqa: E402

DEV = torch.device("cuda:0")
LD = np.longdouble
CHUNK = 4_000_000
CHUNKS = 9                     # x 3 methods = 1.08e8 random tuples
PARAMS = {"sauvola": (0.5, 128.0, 0.0), "niblack": (-0.2, 128.0, 0.0), "wolf": (0.5, 128.0, 17.0)}
# the v5 rules (rule_params as abin_probe_filter takes them): Khurshid {k, N_mode, h w},
# Phansalkar {k, R, p, q} (q >= 0; the configs' q = 10/255 and a steep q)
RULES = {"khurshid0": ("khurshid", (-0.1, 0, 16383.0)), "khurshid0s": ("khurshid", (0.2, 0, 225.0)),
         "khurshid1": ("khurshid", (-0.2, 1, 0.0)), "khurshidN1": ("khurshid", (0.3, 0, 1.0)),
         "phansalkar": ("phansalkar", (0.25, 128.0, 3.0, 10.0 / 255.0)),
         "phansalkar_steep": ("phansalkar", (-0.3, 64.0, -2.0, 0.5)),
         "phansalkar_q0": ("phansalkar", (0.5, 128.0, 1.0, 0.0)),
         # Rais {M S}: the page's product (the bound grows as 1 / (M S)): document pages (M S ~ 7e3),
         # dark / low-contrast pages, and a near-blank one
         "rais_ms7200": ("rais", (7200.0,)), "rais_ms900": ("rais", (900.0,)), "rais_ms40": ("rais", (40.0,)),
         "rais_ms3": ("rais", (3.0,)),
         # Feng {a1, k1, k2, gamma, R} (gamma >= 1), page minimum FENG_L
         "feng_g2": ("feng", (0.12, 0.015, 0.01, 2.0, 128.0)), "feng_g1": ("feng", (0.2, 0.05, 0.02, 1.0, 64.0)),
         "feng_g3": ("feng", (0.1, 0.3, 0.1, 3.0, 100.0))}
FENG_L = 37.0


def t_exact(method, c, d, n, k, R, L):
    V = n.astype(np.int64) * d.astype(np.int64) - c.astype(np.int64) ** 2   # exact (< 2^63)
    assert (V >= 0).all()
    nl = n.astype(LD)
    m = c.astype(LD) / nl
    s = np.sqrt(V.astype(LD) / (nl * nl))
    if method in RULES:
        rule, prm = RULES[method]
        if rule == "feng":
            a1, k1, k2, g, Rf = (LD(v) for v in prm)
            x = s / Rf
            return a1 * m + k1 * x ** (1 + g) * (m - LD(FENG_L)) + k2 * x ** g * LD(FENG_L)
        if rule == "rais":
            # t = m + 0.3 (m s - M S) / max{m s, M S} s  (0/0 -> 0, R16)
            a, b = m * s, LD(prm[0])
            den = np.maximum(a, b)
            f = np.where(den > 0, (a - b) / np.where(den > 0, den, LD(1)), LD(0))
            return m + LD(0.3) * f * s
        if rule == "khurshid":
            # s^2 + m^2 (N - 1) / N = (N n d - c^2) / (N n^2), exact integers (N = h w or n)
            N = n.astype(np.int64) if prm[1] else np.int64(prm[2])
            U = N * n.astype(np.int64) * d.astype(np.int64) - c.astype(np.int64) ** 2
            assert (U >= 0).all()
            return m + LD(prm[0]) * np.sqrt(U.astype(LD) / (LD(1) * N * nl * nl))
        kk, RR, pp, qq = (LD(x) for x in prm)
        return m * (1 + pp * np.exp(-qq * m) + kk * (s / RR - 1))
    k, R, L = LD(k), LD(R), LD(L)
    if method == "sauvola":
        return m * (1 + k * (s / R - 1))
    if method == "niblack":
        return m + k * s
    return m - k * (m - L) * (1 - s / R)


def random_tuples(rng, count):
    ncol = rng.integers(1, 128, count, dtype=np.int64)
    nrow = rng.integers(1, 130, count, dtype=np.int64)
    big = rng.random(count) < 0.5                      # half at the configs' interior sizes
    ncol[big] = rng.choice([15, 31, 32, 61, 63, 101, 127], int(big.sum()))
    nrow[big] = ncol[big]
    nrow = np.minimum(nrow, 129)
    n = ncol * nrow
    c = (rng.random(count) * (255 * n + 1)).astype(np.int64)
    lo = -(-(c * c) // n)                              # ceil(c^2 / n)
    hi = np.minimum(255 * c, 255 * 255 * n)
    d = lo + (rng.random(count) * (hi - lo + 1)).astype(np.int64)
    d = np.minimum(d, hi)
    I = rng.integers(0, 256, count, dtype=np.int64)
    return c, d, ncol, nrow, I


def adversarial_tuples(rng, method, count):
    k, R, L = PARAMS.get(method, (0.0, 1.0, 0.0))
    c, d, ncol, nrow, I = random_tuples(rng, count)
    n = ncol * nrow
    q = count // 6
    # minimum variance (d = ceil(c^2/n)) and constant windows (c = n g, d = n g^2)
    d[:q] = -(-(c[:q] * c[:q]) // n[:q])
    g = rng.integers(0, 256, q)
    c[q:2 * q], d[q:2 * q] = n[q:2 * q] * g, n[q:2 * q] * g * g
    # maximum variance: half 0, half 255
    nn = n[2 * q:3 * q]
    c[2 * q:3 * q] = 255 * (nn // 2)
    d[2 * q:3 * q] = 255 * 255 * (nn // 2)
    # extreme counts
    ncol[3 * q:3 * q + q // 2], nrow[3 * q:3 * q + q // 2] = 1, 1
    ncol[3 * q + q // 2:4 * q], nrow[3 * q + q // 2:4 * q] = 127, 129
    n = ncol * nrow
    c = np.minimum(c, 255 * n)
    lo = -(-(c * c) // n)
    d = np.clip(d, lo, np.minimum(255 * c, 255 * 255 * n))
    # near ties everywhere: I = round(t*)
    t = t_exact(method, c, d, n, k, R, L)
    I = np.clip(np.rint(t.astype(np.float64)), 0, 255).astype(np.int64)
    return c, d, ncol, nrow, I


def run_probe(method, c, d, ncol, nrow, I):
    dev = lambda a, dt: torch.from_numpy(a.astype(dt)).to(DEV)
    args = (dev(c, np.uint32), dev(d, np.uint32), dev(ncol, np.uint32), dev(nrow, np.uint32), dev(I, np.uint8))
    if method in RULES:
        rule, prm = RULES[method]
        e, sv, b = abin.probe_filter(rule, *args, L=FENG_L if rule == "feng" else 0.0, rule_params=prm)
    else:
        k, R, L = PARAMS[method]
        e, sv, b = abin.probe_filter(method, *args, k, R, L)
    return e.cpu().numpy().astype(LD), sv.cpu().numpy().astype(np.float64), b


def check(method, c, d, ncol, nrow, I):
    k, R, L = PARAMS.get(method, (0.0, 1.0, 0.0))
    e, sv, b = run_probe(method, c, d, ncol, nrow, I)
    e_star = I.astype(LD) - t_exact(method, c, d, ncol * nrow, k, R, L)
    err = np.abs(e - e_star).astype(np.float64)
    coarse = b[0]
    if method in RULES and RULES[method][0] == "rais":
        coarse = b[0] + b[2] / RULES[method][1][0]   # the kernel's delta1 + aux1 / (M S)
    assert err.max() <= coarse, (method, err.max(), coarse)
    ratio = err.max() / coarse
    if method == "niblack" or method.startswith(("khurshid", "rais", "feng")):
        # the data-dependent bound the kernel applies to Niblack / Khurshid / Rais / Feng lanes
        with np.errstate(divide="ignore"):
            refined = b[1] + b[2] * np.minimum(b[4], b[3] / sv)
        assert (err <= refined).all(), (method, (err - refined).max())
        ratio = max(ratio, (err / refined).max())
    return ratio


@pytest.mark.parametrize("method", ["sauvola", "niblack", "wolf"])
def test_certified_bound_random(method):
    rng = np.random.default_rng({"sauvola": 1, "niblack": 2, "wolf": 3}[method])
    worst = 0.0
    for _ in range(CHUNKS):
        worst = max(worst, check(method, *random_tuples(rng, CHUNK)))
    assert worst < 1.0
    print(f"{method}: {CHUNKS * CHUNK} random tuples, max |e~ - e*| / bound = {worst:.3g}")


@pytest.mark.parametrize("method", ["sauvola", "niblack", "wolf"])
def test_certified_bound_adversarial(method):
    rng = np.random.default_rng({"sauvola": 11, "niblack": 12, "wolf": 13}[method])
    worst = 0.0
    for _ in range(3):
        worst = max(worst, check(method, *adversarial_tuples(rng, method, 1_000_000)))
    assert worst < 1.0
    print(f"{method}: 3e6 adversarial tuples, max |e~ - e*| / bound = {worst:.3g}")


@pytest.mark.parametrize("method", sorted(RULES))
def test_certified_bound_rules(method):
    """Khurshid, Phansalkar and Rais on v5: the same claim |e~ - e*| <=
    bound for the rule's own residual (moments5.cuh residual2, abin_api.cu
    filter_consts_v5), e* from the exact integers in long double; 1.2e7
    random + 3e6 adversarial tuples per parameter set (11 sets; Rais's bound
    is formed per page from its M S)."""
    rng = np.random.default_rng(100 + sorted(RULES).index(method))
    worst = 0.0
    for _ in range(3):
        worst = max(worst, check(method, *random_tuples(rng, CHUNK)))
    for _ in range(3):
        worst = max(worst, check(method, *adversarial_tuples(rng, method, 1_000_000)))
    assert worst < 1.0
    print(f"{method}: 1.5e7 tuples, max |e~ - e*| / bound = {worst:.3g}")


def test_rule_parameters_outside_v5_are_refused():
    z = torch.zeros(4, dtype=torch.uint32, device=DEV)
    one = torch.ones(4, dtype=torch.uint32, device=DEV)
    I = torch.zeros(4, dtype=torch.uint8, device=DEV)
    with pytest.raises(abin.AbinError):   # q < 0: e^(-q m) unbounded -> exact path only
        abin.probe_filter("phansalkar", z, z, one, one, I, rule_params=(0.25, 128.0, 3.0, -0.1))
