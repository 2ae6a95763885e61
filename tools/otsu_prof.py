"""Per-kernel times of abin_otsu on one config-3 page (torch.profiler)."""
import sys
sys.path.insert(0, '.')
import torch, synth
from torch.profiler import profile, ProfilerActivity
import paper_1905_13038_b200 as ab
x = torch.from_numpy(synth.page(7016, 4960, synth.config_seed(3), stain=True)).cuda()
for _ in range(5): ab.otsu(x)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10): ab.otsu(x)
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        a = agg.setdefault(e.name[:50], [0, 0.0]); a[0] += 1; a[1] += e.device_time_total
for n, (c, tt) in sorted(agg.items(), key=lambda x: -x[1][1]): print(f"{n:50s} n={c} avg={tt / c:.1f} us")
