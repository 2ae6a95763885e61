"""Table-1 rules on one config-3 page (7016 x 4960, 61 x 61): device time per
call (CUDA events, inputs rotated past L2) and the share of pixels decided in
double (counters[1]).  One JSON line per rule."""
import json, sys
sys.path.insert(0, '.')
import torch
from sweep_util import pages_dev, timed  # noqa: E402
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin

RULE_PARAMS = {"feng": (0.85, 0.2, 0.05, 2.0, 64.0), "rais": (), "khurshid": (-0.1, 0), "khurshid_n": (-0.1, 1),
               "phansalkar": (0.25, 128.0, 3.0, 10.0 / 255.0)}
x, nr = pages_dev(1, 7016, 4960, 3, True)
px = 7016 * 4960
for name, prm in RULE_PARAMS.items():
    rule = name.split("_")[0]
    for flags, tag in ((0, ""), (abin.V3_INTERNAL, " v3")):
        ms = timed(lambda k: ab.binarize_rule(rule, x[k, 0], 61, 61, prm, flags=flags), nr, reps=5)
        cnt = torch.zeros(3, dtype=torch.int64, device='cuda')
        ab.binarize_rule(rule, x[0, 0], 61, 61, prm, flags=flags, counters=cnt)
        print(json.dumps({"rule": name + tag, "ms": ms, "gpx_s": px / ms / 1e6,
                          "fp64_share": int(cnt[1]) / px}), flush=True)
