"""Config 5 (one 4096^2 page, 51x51, q = 0.5 / 0.9): time against forced band
counts (ABIN_Q5_BANDS) and the band model's warm-up weight (ABIN_Q5_WU)."""
import json, os, sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tools')
import torch
import paper_1905_13038_b200 as ab
from sweep_util import pages_dev, timed

x, nr = pages_dev(1, 4096, 4096, 5, False)
o = torch.empty((nr, 4096, 4096), dtype=torch.uint8, device='cuda')
for q in (0.5, 0.9):
    os.environ.pop("ABIN_Q5_BANDS", None)
    for wu in ("0.05", "0.1", "0.2", "0.4", "0.8"):
        os.environ["ABIN_Q5_WU"] = wu
        ms = timed(lambda k: ab.quantile(x[k, 0], 51, 51, q, out=o[k]), nr, reps=10)
        print(json.dumps({"q": q, "wu": wu, "ms": ms, "gpx_s": 4096 ** 2 / ms / 1e6}), flush=True)
    os.environ.pop("ABIN_Q5_WU", None)
    for nb in (16, 32, 48, 64, 96, 128, 160, 200, 256, 320, 400):
        os.environ["ABIN_Q5_BANDS"] = str(nb)
        ms = timed(lambda k: ab.quantile(x[k, 0], 51, 51, q, out=o[k]), nr, reps=10)
        print(json.dumps({"q": q, "bands": nb, "ms": ms, "gpx_s": 4096 ** 2 / ms / 1e6}), flush=True)
    os.environ.pop("ABIN_Q5_BANDS", None)
