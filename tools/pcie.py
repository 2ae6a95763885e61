import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device='cuda')
h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2): d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def tm(f):
    torch.cuda.synchronize(); t = time.time(); f(); torch.cuda.synchronize(); return time.time() - t
print("H2D GB/s", n / tm(lambda: d.copy_(h, non_blocking=True)) / 1e9)
print("D2H GB/s", n / tm(lambda: h2.copy_(d2, non_blocking=True)) / 1e9)
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print("both GB/s (sum)", 2 * n / tm(both) / 1e9)
