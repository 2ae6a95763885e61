import sys, os
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin
P = synth.pages(1, 3300, 2550, synth.config_seed(2)); x = torch.zeros((3300, 2560), dtype=torch.uint8, device='cuda')[:, :2550]
x.copy_(torch.from_numpy(P[0]))
for hw in (15, 31):
    cnt = torch.zeros(3, dtype=torch.int64, device='cuda')
    ab.sauvola(x, hw, hw, 0.5, 128.0, counters=cnt, flags=abin.COUNT_STAGES); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); ab.sauvola(x, hw, hw, 0.5, 128.0); b.record(); torch.cuda.synchronize()
    print(os.environ.get("ABIN_V4_BANDS"), hw, cnt.tolist(), a.elapsed_time(b))
