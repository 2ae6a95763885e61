"""Quantile / Bernsen timing on config 5 (one 4096^2 page and the 32-page batch)."""
import os, sys
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
host = synth.pages(32, 4096, 4096, synth.config_seed(5), stain=False)
buf = torch.from_numpy(host).cuda()
def t(f, reps=10):
    for _ in range(5): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
w = torch.zeros(1 << 28, dtype=torch.uint8, device='cuda')   # clocks up before timing
import time
t0 = time.time()
while time.time() - t0 < 1.0: w.add_(1)
res = {}
for name, f, px in [("q0.5 1p", lambda: ab.quantile(buf[0], 51, 51, 0.5), 4096 * 4096),
                    ("q0.1 1p", lambda: ab.quantile(buf[0], 51, 51, 0.1), 4096 * 4096),
                    ("q0.5 32p", lambda: ab.binarize_batched("quantile", buf, 51, 51, 0.5), 32 * 4096 * 4096),
                    ("bernsen 1p", lambda: ab.binarize_batched("bernsen", buf[:1], 51, 51, -1.0), 4096 * 4096)]:
    ms = t(f)
    res[name] = f"{ms:.3f} ms {px / ms / 1e6:.1f} Gpx/s"
print(os.environ.get("ABIN_LIB", "default").split("/")[-1], res, flush=True)
