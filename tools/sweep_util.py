"""Timing helpers shared by tools/sweep.py and tools/rules_perf.py."""
import torch
import synth

L2 = 126e6
def timed(f, n_rot, reps=20):
    for k in range(3): f(k % n_rot)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(reps): f(k % n_rot)
        b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best

def pages_dev(P, H, W, cfg, stain):
    host = synth.pages(P, H, W, synth.config_seed(cfg), stain=stain)
    n_rot = max(1, int(-(-3 * L2 // (2 * P * H * W))))
    pitch = (W + 15) // 16 * 16
    buf = torch.zeros((n_rot, P, H, pitch), dtype=torch.uint8, device='cuda')
    buf[:, :, :, :W] = torch.from_numpy(host).cuda().unsqueeze(0)
    return buf[:, :, :, :W], n_rot

