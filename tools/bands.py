import sys, os, time
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
P, H, W = 64, 7016, 4960
host = synth.pages(P, H, W, synth.config_seed(3), stain=True)
buf = torch.zeros((P, H, W), dtype=torch.uint8, device='cuda'); buf.copy_(torch.from_numpy(host))
out = torch.empty_like(buf)
def t(f, reps=5):
    for _ in range(2): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
w = torch.zeros(1 << 28, dtype=torch.uint8, device='cuda')
t0 = time.time()
while time.time() - t0 < 1.0: w.add_(1)
ms = t(lambda: ab.binarize_batched("sauvola", buf, 61, 61, 0.5, 128.0, out=out))
print(os.environ.get("ABIN_V4_BANDS", "auto"), f"{ms:.3f} ms {P*H*W/ms/1e6:.0f} Gpx/s", flush=True)
