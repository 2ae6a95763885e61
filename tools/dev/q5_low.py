"""Config 5 page at low quantiles: the library default against v5 forced
(ABIN_Q5_ALWAYS) with 1-3 level windows (ABIN_Q5_NW) and the round-1
kernels (Q2_INTERNAL)."""
import json, os, sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tools')
import torch
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin
from sweep_util import pages_dev, timed

x, nr = pages_dev(1, 4096, 4096, 5, False)
o = torch.empty((nr, 4096, 4096), dtype=torch.uint8, device='cuda')
qs = [float(a) for a in sys.argv[1:]] or [0.1, 0.15, 0.2]
for q in qs:
    for mode in ("default", "round1", "v5nw1", "v5nw2", "v5nw3"):
        for k in ("ABIN_Q5_ALWAYS", "ABIN_Q5_NW"):
            os.environ.pop(k, None)
        if mode.startswith("v5"):
            os.environ["ABIN_Q5_ALWAYS"] = "1"
            os.environ["ABIN_Q5_NW"] = mode[-1]
        fl = abin.Q2_INTERNAL if mode == "round1" else 0
        ms = timed(lambda k: ab.quantile(x[k, 0], 51, 51, q, out=o[k], flags=fl), nr, reps=5)
        print(json.dumps({"q": q, "mode": mode, "ms": ms, "gpx_s": 4096 ** 2 / ms / 1e6}), flush=True)
