"""Per-kernel device durations (torch.profiler / CUPTI) of one binarize call
on a config-3-like 16-page batch: which launches a call makes and their times."""
import os, sys
sys.path.insert(0, '.')
import torch, synth
from torch.profiler import profile, ProfilerActivity
import paper_1905_13038_b200 as ab
P, H, W = 16, 7016, 4960
host = synth.pages(P, H, W, synth.config_seed(3), stain=True)
buf = torch.zeros((P, H, W), dtype=torch.uint8, device='cuda'); buf.copy_(torch.from_numpy(host))
method = sys.argv[1] if len(sys.argv) > 1 else "sauvola"
k = {"sauvola": 0.5, "niblack": -0.2, "wolf": 0.5}[method]
f = lambda: ab.binarize_batched(method, buf, 61, 61, k, 128.0)
for _ in range(5): f()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10): f()
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        a = agg.setdefault(e.name[:60], [0, 0.0])
        a[0] += 1; a[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
tag = os.environ.get("ABIN_LIB", "default").split("/")[-1]
# timeline of the last two calls: start offsets / durations / gaps (us)
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
last = evs[-12:]
t0 = last[0].time_range.start
prev_end = None
for e in last:
    gap = (e.time_range.start - prev_end) if prev_end is not None else 0
    print(f"{tag} {method} t={e.time_range.start - t0:9.1f} dur={e.time_range.end - e.time_range.start:8.1f} gap={gap:6.1f} {e.name[:50]}")
    prev_end = e.time_range.end
for n, (c, tt) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{tag} {method} {n:60s} n={c:3d} avg={tt / c:9.1f} us")
cnt = torch.zeros(3, dtype=torch.int64, device='cuda')
from paper_1905_13038_b200 import abin as _abin
ab.binarize_batched(method, buf, 61, 61, k, 128.0, counters=cnt, flags=_abin.COUNT_STAGES)
torch.cuda.synchronize()
print(tag, method, "near ties / fp64 / stage-2 pixels:", cnt.tolist(), "of", buf.numel())
