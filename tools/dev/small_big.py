"""Does the tile kernel (small.cuh) beat the streaming kernels on larger
single pages?  (dev tool)  Run once per ABIN_SMALL_PX setting: the config-2
page and an A4 page at small windows, device time per call."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import latency  # noqa: E402

if __name__ == "__main__":
    for (H, W) in ((1024, 1024), (2048, 2048), (3300, 2550), (7016, 4960)):
        for hw in (15, 31, 63):
            r = latency.measure(H, W, hw, hw, n=30)
            r["ABIN_SMALL_PX"] = os.environ.get("ABIN_SMALL_PX", "default")
            print(json.dumps(r), flush=True)
