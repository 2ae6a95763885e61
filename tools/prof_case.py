"""Run one BASELINE config's kernel a few times (for ncu captures)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import synth
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin
cfg = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
npages = int(sys.argv[3]) if len(sys.argv) > 3 else None
C = {1: (1, 512, 512, 32, 32, 'sauvola', 0.5, False, False), 2: (1, 3300, 2550, 63, 63, 'sauvola', 0.5, False, False),
     3: (64, 7016, 4960, 61, 61, 'sauvola', 0.5, False, True), 4: (1, 32768, 32768, 101, 101, 'sauvola', 0.34, True, False),
     5: (1, 4096, 4096, 51, 51, 'quantile', 0.5, False, False)}
P, H, W, h, w, method, k, packed, stain = C[cfg]
if npages: P = npages
pitch = (W + 15) // 16 * 16
host = synth.pages(P, H, W, synth.config_seed(cfg), stain=stain)
buf = torch.zeros((P, H, pitch), dtype=torch.uint8, device='cuda')
buf[:, :, :W] = torch.from_numpy(host).cuda()
x = buf[:, :, :W]
flags = abin.FORCE_U64_SQ if cfg == 4 else 0
for _ in range(reps):
    if method == 'quantile':
        ab.quantile(x[0], h, w, k)
    else:
        ab.binarize_batched(method, x, h, w, k, 128.0, packed=packed, flags=flags)
torch.cuda.synchronize()
print('ok', cfg, P, H, W)
