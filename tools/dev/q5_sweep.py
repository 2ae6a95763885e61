"""v5 quantile: config-5 page time vs band count and window count (dev tool)."""
import os, sys
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
I = synth.page(4096, 4096, synth.config_seed(5))
xs = [torch.from_numpy(I).cuda() for _ in range(4)]
def timeit(q, reps=10):
    for k in range(3): ab.binarize_batched("quantile", xs[k % 4].unsqueeze(0), 51, 51, q)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(reps): ab.binarize_batched("quantile", xs[k % 4].unsqueeze(0), 51, 51, q)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for q in (0.5, 0.9, 0.1):
    cnt = torch.zeros(3, dtype=torch.int64, device='cuda')
    ab.binarize_batched("quantile", xs[0].unsqueeze(0), 51, 51, q, counters=cnt)
    ms = timeit(q)
    print(f"default q={q}: {ms:.3f} ms {I.size / ms / 1e6:.1f} Gpx/s exact {int(cnt[1])}", flush=True)
for bands in ("8", "16", "32", "64", "128", "241"):
    os.environ["ABIN_Q5_BANDS"] = bands
    ms = timeit(0.5)
    print(f"bands {bands} q=0.5: {ms:.3f} ms {I.size / ms / 1e6:.1f} Gpx/s", flush=True)
os.environ.pop("ABIN_Q5_BANDS")
P = torch.from_numpy(synth.pages(32, 4096, 4096, synth.config_seed(5))).cuda()
for k in range(2): ab.binarize_batched("quantile", P, 51, 51, 0.5)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for k in range(3): ab.binarize_batched("quantile", P, 51, 51, 0.5)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
print(f"5b (32 pages) q=0.5: {ms:.3f} ms {P.numel() / ms / 1e6:.1f} Gpx/s", flush=True)
