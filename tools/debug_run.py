import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle
import paper_1905_13038_b200 as ab
mode, H, W, h, w = sys.argv[1], *map(int, sys.argv[2:6])
I = synth.page(H, W, synth.config_seed(1))
x = torch.from_numpy(I).cuda()
flags = (1 << 30) if mode == "notma" else 0
t = time.time()
m = ab.sauvola(x, h, w, 0.5, 128.0, flags=flags)
try:
    torch.cuda.synchronize()
    got = m.cpu().numpy()
    ref = oracle.binarize("sauvola", I, h, w, 0.5, 128.0)
    print(mode, H, W, h, w, "time", time.time() - t, "mismatch", int((got != ref).sum()), "of", ref.size)
except Exception as e:
    print(mode, H, W, h, w, "ERR after", time.time() - t, str(e)[:60])
