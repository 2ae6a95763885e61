"""Config 2 page: time vs forced band count (ABIN_V4_BANDS) per window size."""
import os, sys
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
def t(f, reps=30):
    for _ in range(5): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
H, W = 3300, 2550
buf = torch.zeros((H, 2560), dtype=torch.uint8, device='cuda'); buf[:, :W] = torch.from_numpy(synth.page(H, W, 9)).cuda()
x = buf[:, :W]
o = torch.empty((H, W), dtype=torch.uint8, device='cuda')
for hw in (31, 63, 127, 255):
    res = []
    for nb in ("auto", 8, 16, 32, 64, 100, 150, 206):
        if nb == "auto": os.environ.pop("ABIN_V4_BANDS", None)
        else: os.environ["ABIN_V4_BANDS"] = str(nb)
        res.append(f"{nb}:{t(lambda: ab.sauvola(x, hw, hw, 0.5, 128.0, out=o)):.0f}")
    print(f"w={hw}", " ".join(res), flush=True)
