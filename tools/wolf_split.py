import sys
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
P, H, W = 16, 7016, 4960
host = synth.pages(P, H, W, synth.config_seed(3), stain=True)
buf = torch.zeros((P, H, 4960), dtype=torch.uint8, device='cuda'); buf.copy_(torch.from_numpy(host))
def t(f, reps=10):
    for _ in range(5): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
w = torch.zeros(1 << 28, dtype=torch.uint8, device='cuda')
for _ in range(200): w.add_(1)
print("global_min", t(lambda: ab.global_min(buf)))
print("wolf L=-1 ", t(lambda: ab.binarize_batched("wolf", buf, 61, 61, 0.5, 128.0)))
print("wolf L=20 ", t(lambda: ab.binarize_batched("wolf", buf, 61, 61, 0.5, 128.0, L=20)))
print("sauvola   ", t(lambda: ab.binarize_batched("sauvola", buf, 61, 61, 0.5, 128.0)))
print("niblack   ", t(lambda: ab.binarize_batched("niblack", buf, 61, 61, -0.2, 128.0)))
