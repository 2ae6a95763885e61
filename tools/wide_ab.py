import sys
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
for hw in (15, 31, 63, 127, 191, 255):
    a = t(lambda: ab.sauvola(x, hw, hw, 0.5, 128.0, out=o))
    b = t(lambda: ab.sauvola(x, hw, hw, 0.5, 128.0, out=o, flags=1 << 28))
    m1 = ab.sauvola(x, hw, hw, 0.5, 128.0); m2 = ab.sauvola(x, hw, hw, 0.5, 128.0, flags=1 << 28)
    print(f"w={hw}: v4 {a:.1f} us, wide {b:.1f} us, equal {bool(torch.equal(m1, m2))}", flush=True)
