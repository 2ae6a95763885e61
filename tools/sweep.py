"""Config 2's window sweep (cost independent of h, w: PAPER.md:138, 180) and a
results table for every config / method, device-timed with CUDA events on
inputs rotated past L2.  Writes one JSON line per measurement to stdout."""
import json, sys, time
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin

L2 = 126e6
def timed(f, n_rot, reps=20):
    for k in range(3): f(k % n_rot)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(reps): f(k % n_rot)
        b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best

def pages_dev(P, H, W, cfg, stain):
    host = synth.pages(P, H, W, synth.config_seed(cfg), stain=stain)
    n_rot = max(1, int(-(-3 * L2 // (2 * P * H * W))))
    pitch = (W + 15) // 16 * 16
    buf = torch.zeros((n_rot, P, H, pitch), dtype=torch.uint8, device='cuda')
    buf[:, :, :, :W] = torch.from_numpy(host).cuda().unsqueeze(0)
    return buf[:, :, :, :W], n_rot

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
