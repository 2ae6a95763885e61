"""A/B of the moments kernels (v3 4-warp CTAs vs v4 warp CTAs) + stage counters, on BASELINE shapes."""
import sys
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin

def run(tag, P, H, W, h, w, method, k, packed, flags, stain, seedcfg, reps=5):
    pitch = (W + 15) // 16 * 16
    host = synth.pages(P, H, W, synth.config_seed(seedcfg), stain=stain)
    buf = torch.zeros((P, H, pitch), dtype=torch.uint8, device='cuda')
    buf[:, :, :W] = torch.from_numpy(host).cuda()
    x = buf[:, :, :W]
    cnt = torch.zeros(3, dtype=torch.int64, device='cuda')
    outs = {}
    for name, fl in (("v3", flags | abin.V3_INTERNAL), ("v4", flags)):
        f = lambda: ab.binarize_batched(method, x, h, w, k, 128.0, packed=packed, flags=fl | abin.COUNT_STAGES, counters=cnt)
        o = f(); torch.cuda.synchronize(); outs[name] = o.clone(); cnt.zero_()
        for _ in range(10): f()
        torch.cuda.synchronize(); cnt.zero_()
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / reps)
        ms = best
        c = (cnt / reps).tolist()
        print(f"{tag} {name}: {ms:.3f} ms {P*H*W/ms/1e6:.1f} Gpx/s  near_ties {c[0]:.0f} fp64 {c[1]:.0f} stage2 {c[2]:.0f} ({c[2]/(P*H*W):.2e}/px)", flush=True)
    print(f"{tag} v3==v4: {torch.equal(outs['v3'], outs['v4'])}", flush=True)

# warm the GPU clocks up for ~1 s before timing anything
_w = torch.zeros(1 << 28, dtype=torch.uint8, device='cuda')
_t = __import__('time').time()
while __import__('time').time() - _t < 1.5:
    _w.add_(1)
torch.cuda.synchronize()
run("cfg3-sauvola", 16, 7016, 4960, 61, 61, "sauvola", 0.5, False, 0, True, 3)
run("cfg3-niblack", 16, 7016, 4960, 61, 61, "niblack", -0.2, False, 0, True, 3)
run("cfg3-wolf", 16, 7016, 4960, 61, 61, "wolf", 0.5, False, 0, True, 3)
run("cfg4", 1, 32768, 32768, 101, 101, "sauvola", 0.34, True, abin.FORCE_U64_SQ, False, 4)
#run("cfg2-15", 1, 3300, 2550, 15, 15, "sauvola", 0.5, False, 0, False, 2)
#run("cfg2-255", 1, 3300, 2550, 255, 255, "sauvola", 0.5, False, 0, False, 2)
