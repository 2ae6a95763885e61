import sys
sys.path.insert(0, '.')
import numpy as np, torch, synth, oracle
import paper_1905_13038_b200 as ab
P, H, W = 3, 230, 333
pages = synth.pages(P, H, W, synth.config_seed(3), stain=True)
pages[1, 100:140] = 200
for pg in range(P):
    J = pages[pg]
    ref, lo, hi = oracle.bernsen(J, 31, 25, 15)
    whole = ab.bernsen(torch.from_numpy(J).cuda(), 31, 25, 15).cpu().numpy()
    parts = []
    R = 58
    for r0 in range(0, H, R):
        r1 = min(H, r0 + R)
        top, bot = min(15, r0), min(15, H - r1)
        held = torch.from_numpy(np.ascontiguousarray(J[r0 - top:r1 + bot])).cuda()
        parts.append(ab.binarize_band("bernsen", held, r0, H, top, bot, 31, 25, 15.0).cpu().numpy())
    band = np.concatenate(parts)
    print(pg, "whole==oracle", np.array_equal(whole, ref), "band==oracle", np.array_equal(band, ref),
          "diff rows", np.unique(np.nonzero(band != ref)[0])[:20])
