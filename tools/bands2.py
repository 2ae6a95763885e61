import sys, os, time
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
w = torch.zeros(1 << 28, dtype=torch.uint8, device='cuda')
t0 = time.time()
while time.time() - t0 < 1.0: w.add_(1)
if sys.argv[1] == "c2":
    P = synth.pages(1, 3300, 2550, synth.config_seed(2)); x = torch.zeros((3300, 2560), dtype=torch.uint8, device='cuda')[:, :2550]
    x.copy_(torch.from_numpy(P[0]))
    res = []
    for hw in (15, 31, 63, 127, 255):
        ms = t(lambda: ab.sauvola(x, hw, hw, 0.5, 128.0))
        res.append(f"{hw}:{ms*1000:.0f}us")
    print(os.environ.get("ABIN_V4_BANDS", "auto"), " ".join(res), flush=True)
else:
    P = synth.pages(64, 7016, 4960, synth.config_seed(3), stain=True); x = torch.from_numpy(P).cuda()
    print("wolf L=-1", t(lambda: ab.binarize_batched("wolf", x, 61, 61, 0.5, 128.0), 5))
    print("wolf L=20", t(lambda: ab.binarize_batched("wolf", x, 61, 61, 0.5, 128.0, L=20), 5))
    print("gmin", t(lambda: ab.global_min(x), 5))
