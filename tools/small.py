"""Small single pages: v4 + fixup (default) vs the v3 kernel alone (V3_INTERNAL)."""
import sys
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin
def t(f, reps=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
for (H, W, hw) in [(512, 512, 32), (1024, 1024, 31), (2048, 2048, 61), (3300, 2550, 63), (7016, 4960, 61)]:
    x = torch.from_numpy(synth.page(H, W, 7)).cuda()
    o = torch.empty_like(x)
    a = t(lambda: ab.sauvola(x, hw, hw, 0.5, 128.0, out=o))
    b = t(lambda: ab.sauvola(x, hw, hw, 0.5, 128.0, out=o, flags=abin.V3_INTERNAL))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ab.sauvola(x, hw, hw, 0.5, 128.0, out=o)
    c = t(lambda: g.replay())
    print(f"{H}x{W} w={hw}: v4+fixup {a:.1f} us, v3 {b:.1f} us, v4 graph-replayed {c:.1f} us", flush=True)
