"""Config 1 and the tile kernel's larger pages, device time per call (dev
tool; ABIN_LIB selects the build)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import latency  # noqa: E402

if __name__ == "__main__":
    for (H, W, h, w) in ((512, 512, 32, 32), (512, 512, 61, 61), (1024, 1024, 15, 15), (1024, 1024, 32, 32),
                         (1024, 1024, 63, 63), (1400, 1400, 32, 32)):
        r = latency.measure(H, W, h, w, n=100)
        r["lib"] = os.path.basename(os.environ.get("ABIN_LIB", "libabin.so"))
        print(json.dumps(r), flush=True)
