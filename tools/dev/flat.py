"""Config-2 window sweep on a 16-page batch of letter pages (one
binarize_batched launch per window): used under ncu to split each window's
time between k_mom5 / k_mom4 and the exact-fixup kernel."""
import sys
sys.path.insert(0, '.')
import torch
import synth
import paper_1905_13038_b200 as ab

P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
page = synth.page(3300, 2550, synth.config_seed(2, 0))
x = torch.zeros((P, 3300, 2560), dtype=torch.uint8, device='cuda')
x[:, :, :2550] = torch.from_numpy(page).cuda()
o = torch.empty((P, 3300, 2550), dtype=torch.uint8, device='cuda')
cnt = torch.zeros(2, dtype=torch.int64, device='cuda')
for hw in (15, 31, 63, 127, 255):
    cnt.zero_()
    ab.binarize_batched("sauvola", x[:, :, :2550], hw, hw, 0.5, 128.0, out=o, counters=cnt)
    torch.cuda.synchronize()
    print(hw, cnt.tolist(), flush=True)
