"""Exact-queue share of the v5 quantile kernel on config-5 pages, per q and window count."""
import os, sys
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
I = synth.page(4096, 4096, synth.config_seed(5))
x = torch.from_numpy(I).cuda()
for nw in ("1", "2", "3"):
    os.environ["ABIN_Q5_NW"] = nw
    for q in (0.5, 0.1, 0.9):
        cnt = torch.zeros(3, dtype=torch.int64, device='cuda')
        ab.binarize_batched("quantile", x.unsqueeze(0), 51, 51, q, counters=cnt)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3): ab.binarize_batched("quantile", x.unsqueeze(0), 51, 51, q)
        a.record()
        for _ in range(10): ab.binarize_batched("quantile", x.unsqueeze(0), 51, 51, q)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"nw={nw} q={q}: exact {int(cnt[1])} ({int(cnt[1]) / I.size:.2e}), {ms:.3f} ms, {I.size / ms / 1e6:.1f} Gpx/s", flush=True)
os.environ.pop("ABIN_Q5_NW")
for q in (0.5, 0.1, 0.9):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ab.binarize_batched("quantile", x.unsqueeze(0), 51, 51, q, flags=ab.abin.Q2_INTERNAL)
    a.record()
    for _ in range(5): ab.binarize_batched("quantile", x.unsqueeze(0), 51, 51, q, flags=ab.abin.Q2_INTERNAL)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"round-1 kernel q={q}: {ms:.3f} ms, {I.size / ms / 1e6:.1f} Gpx/s", flush=True)
