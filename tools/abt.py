"""A/B timing of library variants on config-3-like batches (16 pages), per method."""
import sys, os, time
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
P, H, W = 16, 7016, 4960
host = synth.pages(P, H, W, synth.config_seed(3), stain=True)
buf = torch.zeros((P, H, W), dtype=torch.uint8, device='cuda'); buf.copy_(torch.from_numpy(host))
g = synth.page(32768, 32768, synth.config_seed(4)); gb = torch.from_numpy(g).cuda(); del g
def t(f, reps=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best
w = torch.zeros(1 << 28, dtype=torch.uint8, device='cuda')
t0 = time.time()
while time.time() - t0 < 1.0: w.add_(1)
res = {}
for name, f in [("sauvola", lambda: ab.binarize_batched("sauvola", buf, 61, 61, 0.5, 128.0)),
                ("niblack", lambda: ab.binarize_batched("niblack", buf, 61, 61, -0.2, 128.0)),
                ("wolf", lambda: ab.binarize_batched("wolf", buf, 61, 61, 0.5, 128.0)),
                ("cfg4", lambda: ab.sauvola(gb, 101, 101, 0.34, 128.0, packed=True, flags=1))]:
    ms = t(f)
    px = gb.numel() if name == "cfg4" else buf.numel()
    res[name] = f"{ms:.3f} ms {px / ms / 1e6:.0f} Gpx/s"
print(os.environ.get("ABIN_LIB", "default").split("/")[-1], res, flush=True)
