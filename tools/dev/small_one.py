"""One tile-kernel call on a 1024^2 page at 32 x 32 (dev tool: the ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
import paper_1905_13038_b200 as ab  # noqa: E402

x = torch.from_numpy(synth.page(1024, 1024, synth.config_seed(2, 0))).to("cuda:0")
for _ in range(3):
    m = ab.sauvola(x, 32, 32, 0.5, 128.0)
torch.cuda.synchronize()
print(int(m.sum()))
