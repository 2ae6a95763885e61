"""Bernsen timing (dev): the window-independent kernels vs the histogram
kernels on a config-5 page (4096^2) and the config-2 window sweep."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
import paper_1905_13038_b200 as ab  # noqa: E402
from paper_1905_13038_b200 import abin  # noqa: E402


def t(H, W, h, w, flags=0, n=20, pages=1):
    x = torch.from_numpy(synth.pages(pages, H, W, synth.config_seed(5, 0))).cuda()
    out = torch.empty_like(x)
    for _ in range(3):
        ab.binarize_batched("bernsen", x, h, w, -1.0, out=out, flags=flags)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(1e8))
    a.record()
    for _ in range(n):
        ab.binarize_batched("bernsen", x, h, w, -1.0, out=out, flags=flags)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / n * 1e3
    return {"H": H, "W": W, "pages": pages, "h": h, "w": w, "flags": flags, "us": round(us, 1),
            "gpx_s": round(pages * H * W / us / 1e3, 1)}


if __name__ == "__main__":
    print(json.dumps(t(4096, 4096, 51, 51)))
    print(json.dumps(t(4096, 4096, 51, 51, flags=abin.Q2_INTERNAL, n=5)))
    print(json.dumps(t(4096, 4096, 51, 51, pages=8, n=10)))
    for hw in (15, 31, 63, 127, 255):
        print(json.dumps(t(3300, 2550, hw, hw)))
