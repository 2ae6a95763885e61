import os, sys
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
host = synth.pages(4, 4096, 4096, synth.config_seed(5), stain=False)
buf = torch.from_numpy(host).cuda()
def t(f, reps=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for rep in range(2):
    for pg in range(4):
        for q in (0.5, 0.1, 0.9):
            ms = t(lambda: ab.quantile(buf[pg], 51, 51, q))
            print(os.environ.get("ABIN_LIB","").split("/")[-1], rep, pg, q, f"{ms:.3f} ms", flush=True)
