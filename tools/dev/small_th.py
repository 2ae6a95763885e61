"""Tile height 16 vs 32 of the small-call kernel (dev tool; ABIN_SMALL_TH32 =
the tiles-per-SM threshold, a large value keeps 16-row tiles)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import latency  # noqa: E402

if __name__ == "__main__":
    for (H, W) in ((512, 512), (1024, 1024), (1400, 1400), (2048, 2048)):
        for hw in (15, 32, 63):
            r = latency.measure(H, W, hw, hw, n=50)
            r["ABIN_SMALL_TH32"] = os.environ.get("ABIN_SMALL_TH32", "default")
            print(json.dumps(r), flush=True)
