"""Config 2's window sweep (cost independent of h, w: PAPER.md:138, 180) and a
results table for every config / method, device-timed with CUDA events on
inputs rotated past L2.  Writes one JSON line per measurement to stdout."""
import json, sys, time
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin

from sweep_util import L2, pages_dev, timed  # noqa: E402

w = torch.zeros(1 << 28, dtype=torch.uint8, device='cuda')
t0 = time.time()
while time.time() - t0 < 1.0: w.add_(1)
peak = 6532.9
# config 2 window sweep
x, nr = pages_dev(1, 3300, 2550, 2, False)
outs = torch.empty((nr, 3300, 2550), dtype=torch.uint8, device='cuda')
for hw in (15, 31, 63, 127, 255):
    ms = timed(lambda k: ab.sauvola(x[k, 0], hw, hw, 0.5, 128.0, out=outs[k]), nr)
    px = 3300 * 2550
    print(json.dumps({"sweep": "config2", "h": hw, "w": hw, "ms": ms, "gpx_s": px / ms / 1e6,
                      "frac": 2 * px / ms / 1e6 / peak}), flush=True)
# config 3 methods (64 pages)
x, nr = pages_dev(64, 7016, 4960, 3, True)
out = torch.empty((64, 7016, 4960), dtype=torch.uint8, device='cuda')
for method, k in (("sauvola", 0.5), ("niblack", -0.2), ("wolf", 0.5)):
    ms = timed(lambda q: ab.binarize_batched(method, x[q], 61, 61, k, 128.0, out=out), nr, reps=5)
    px = 64 * 7016 * 4960
    print(json.dumps({"config": 3, "method": method, "ms": ms, "gpx_s": px / ms / 1e6,
                      "frac": 2 * px / ms / 1e6 / peak}), flush=True)
del x, out
# config 5 quantiles and Bernsen
x, nr = pages_dev(1, 4096, 4096, 5, False)
o5 = torch.empty((nr, 4096, 4096), dtype=torch.uint8, device='cuda')
for q in (0.5, 0.1, 0.9):
    ms = timed(lambda k: ab.quantile(x[k, 0], 51, 51, q, out=o5[k]), nr, reps=5)
    print(json.dumps({"config": 5, "method": f"quantile q={q}", "ms": ms, "gpx_s": 4096 * 4096 / ms / 1e6,
                      "frac": 2 * 4096 * 4096 / ms / 1e6 / peak}), flush=True)
ms = timed(lambda k: ab.bernsen(x[k, 0], 51, 51, -1, out=o5[k]), nr, reps=5)
print(json.dumps({"config": 5, "method": "bernsen", "ms": ms, "gpx_s": 4096 * 4096 / ms / 1e6}), flush=True)
# config 5b: the 32-page quantile batch
xb = torch.from_numpy(synth.pages(32, 4096, 4096, synth.config_seed(5), stain=False)).cuda()
ms = timed(lambda k: ab.binarize_batched("quantile", xb, 51, 51, 0.5), 1, reps=3)
print(json.dumps({"config": "5b", "method": "quantile q=0.5, 32 pages", "ms": ms, "gpx_s": 32 * 4096 * 4096 / ms / 1e6,
                  "frac": 2 * 32 * 4096 * 4096 / ms / 1e6 / peak}), flush=True)
del xb
# config 1 (one 512^2 page, 32x32, inputs rotated past L2)
x, nr = pages_dev(1, 512, 512, 1, False)
o1 = torch.empty((nr, 512, 512), dtype=torch.uint8, device='cuda')
ms = timed(lambda k: ab.sauvola(x[k, 0], 32, 32, 0.5, 128.0, out=o1[k]), nr, reps=50)
print(json.dumps({"config": 1, "method": "sauvola", "ms": ms, "gpx_s": 512 * 512 / ms / 1e6}), flush=True)
# config 4 (32768^2, 101x101, forced u64 square sums, bit mask)
g = torch.from_numpy(synth.page(32768, 32768, synth.config_seed(4))).cuda()
ms = timed(lambda k: ab.sauvola(g, 101, 101, 0.34, 128.0, packed=True, flags=abin.FORCE_U64_SQ), 1, reps=5)
print(json.dumps({"config": 4, "method": "sauvola bits u64", "ms": ms, "gpx_s": 32768 ** 2 / ms / 1e6,
                  "frac": 1.125 * 32768 ** 2 / ms / 1e6 / peak}), flush=True)
# the same without forcing: 255^2 h w < 2^32 at 101 x 101, so the paper's own rule keeps u32 sums (v5)
ms = timed(lambda k: ab.sauvola(g, 101, 101, 0.34, 128.0, packed=True), 1, reps=5)
print(json.dumps({"config": 4, "method": "sauvola bits u32 (v5)", "ms": ms, "gpx_s": 32768 ** 2 / ms / 1e6,
                  "frac": 1.125 * 32768 ** 2 / ms / 1e6 / peak}), flush=True)
del g
# NEXT rows on one config-3 page: Table 1 rules and Otsu
x, nr = pages_dev(1, 7016, 4960, 3, True)
RULE_PARAMS = {"feng": (0.85, 0.2, 0.05, 2.0, 64.0), "rais": (), "khurshid": (-0.1, 0),
               "phansalkar": (0.25, 128.0, 3.0, 10.0 / 255.0)}   # as in tests/test_gpu_parity.py
for rule in ("feng", "rais", "khurshid", "phansalkar"):
    ms = timed(lambda k: ab.binarize_rule(rule, x[k, 0], 61, 61, RULE_PARAMS[rule]), nr, reps=5)
    print(json.dumps({"next": rule, "ms": ms, "gpx_s": 7016 * 4960 / ms / 1e6}), flush=True)
ms = timed(lambda k: ab.otsu(x[k, 0]), nr, reps=5)
print(json.dumps({"next": "otsu", "ms": ms, "gpx_s": 7016 * 4960 / ms / 1e6}), flush=True)
# NEXT #3: Wolf with the adaptive R (max s: two v5 passes + exact candidates; one host sync per page)
ms = timed(lambda k: ab.wolf_adaptive(x[k, 0], 61, 61, 0.5), nr, reps=5)
print(json.dumps({"next": "wolf_adaptive", "ms": ms, "gpx_s": 7016 * 4960 / ms / 1e6}), flush=True)
