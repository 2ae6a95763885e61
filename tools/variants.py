"""Time kernel variants on synthetic pages (CUDA events), for quick A/B checks."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import synth
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin

def run(P, H, W, h, w, k, packed, flags, reps=5, method='sauvola', pad=0, seedcfg=4, stain=False):
    pitch = (W + 15) // 16 * 16 + pad
    host = synth.pages(P, H, W, synth.config_seed(seedcfg), stain=stain)
    buf = torch.zeros((P, H, pitch), dtype=torch.uint8, device='cuda')
    buf[:, :, :W] = torch.from_numpy(host).cuda()
    x = buf[:, :, :W]
    cnt = torch.zeros(2, dtype=torch.int64, device='cuda')
    f = lambda: ab.binarize_batched(method, x, h, w, k, 128.0, packed=packed, flags=flags, counters=cnt)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"seed{seedcfg} stain{stain} pad{pad} P{P} {H}x{W} h{h} w{w} k{k} packed{packed} flags{flags} {method}: {ms:.3f} ms  {P*H*W/ms/1e6:.1f} Gpx/s  cnt {cnt.tolist()}", flush=True)

for spec in sys.argv[1:]:
    P, H, W, h, w, k, packed, flags, pad, seedcfg, stain = (spec.split(',') + ['0', '4', '0'][len(spec.split(',')) - 8:])[:11]
    run(int(P), int(H), int(W), int(h), int(w), float(k), packed == '1', int(flags), pad=int(pad), seedcfg=int(seedcfg), stain=stain == '1')
