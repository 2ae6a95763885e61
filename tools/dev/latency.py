"""Small-page latency breakdown (dev tool): host time per call, device time
back to back, device time with the host run ahead (a sleep kernel first), and
the CUDA-graph replay time, for config 1 and the config-2 window sweep."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
import paper_1905_13038_b200 as ab  # noqa: E402


def measure(H, W, h, w, n=50, method="sauvola", q=0.5):
    dev = torch.device("cuda:0")
    pitch = (W + 15) // 16 * 16
    xs = torch.zeros((8, H, pitch), dtype=torch.uint8, device=dev)
    xs[:, :, :W] = torch.from_numpy(synth.page(H, W, synth.config_seed(2, 0))).to(dev)
    x = xs[:, :, :W]
    out = torch.empty((8, H, W), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()

    def call(i):
        if method == "quantile":
            ab.quantile(x[i % 8], h, w, q, out=out[i % 8])
        else:
            ab.sauvola(x[i % 8], h, w, 0.5, 128.0, out=out[i % 8])
    for i in range(5):
        call(i)
    torch.cuda.synchronize()
    # host time per call
    t0 = time.perf_counter()
    for i in range(n):
        call(i)
    host_us = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    # back to back (events)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for i in range(n):
        call(i)
    b.record(st)
    torch.cuda.synchronize()
    b2b_us = a.elapsed_time(b) / n * 1e3
    # host runs ahead behind a sleep kernel: device time only
    torch.cuda._sleep(int(2e8))
    a.record(st)
    for i in range(n):
        call(i)
    b.record(st)
    torch.cuda.synchronize()
    dev_us = a.elapsed_time(b) / n * 1e3
    # CUDA graph of n calls
    graph_us = None
    try:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(st)
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for i in range(n):
                    call(i)
        st.wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        a.record(st)
        g.replay()
        b.record(st)
        torch.cuda.synchronize()
        graph_us = a.elapsed_time(b) / n * 1e3
    except Exception as e:  # noqa: BLE001
        graph_us = f"capture failed: {e}"[:200]
    return {"method": method, "H": H, "W": W, "h": h, "w": w, "host_us": round(host_us, 2), "b2b_us": round(b2b_us, 2),
            "dev_us": round(dev_us, 2), "graph_us": graph_us if isinstance(graph_us, str) else round(graph_us, 2),
            "gpx_dev": round(H * W / dev_us / 1e3, 1)}


if __name__ == "__main__":
    if "--quantile" in sys.argv:
        for q in (0.5, 0.1, 0.9):
            print(json.dumps(measure(4096, 4096, 51, 51, n=10, method="quantile", q=q)))
        sys.exit(0)
    rows = [measure(512, 512, 32, 32)]
    for hw in (15, 31, 63, 127, 255):
        rows.append(measure(3300, 2550, hw, hw))
    for r in rows:
        print(json.dumps(r))
