"""Stage-2 (exact fixup) pixel counts against page width / window: which
lanes does the fp32 filter queue (ABIN_COUNT_STAGES)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import synth
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin

for W in (2550, 2560, 2551, 2553, 2558, 2400, 2401):
    for hw in (9, 15, 31):
        for v4 in (0, 1):
            I = synth.page(256, W, 1234)
            pitch = (W + 15) // 16 * 16
            buf = torch.zeros((256, pitch), dtype=torch.uint8, device='cuda')
            buf[:, :W] = torch.from_numpy(I).cuda()
            cnt = torch.zeros(3, dtype=torch.int64, device='cuda')
            ab.sauvola(buf[:, :W], hw, hw, 0.5, 128.0, counters=cnt,
                       flags=abin.COUNT_STAGES | (abin.V4_INTERNAL if v4 else 0))
            torch.cuda.synchronize()
            print(W, hw, "v4" if v4 else "v5", cnt.tolist(), flush=True)
