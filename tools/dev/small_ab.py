"""A/B of the small-call kernel (dev tool): device time per call of config 1
and a few other small pages, printed as JSON lines; run once per library
(ABIN_LIB selects the build)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import latency  # noqa: E402

if __name__ == "__main__":
    for (H, W, h, w) in ((512, 512, 32, 32), (512, 512, 15, 15), (512, 512, 61, 61), (300, 700, 32, 32),
                         (512, 1024, 32, 32)):
        r = latency.measure(H, W, h, w, n=200)
        r["lib"] = os.path.basename(os.environ.get("ABIN_LIB", "libabin.so"))
        print(json.dumps(r))
