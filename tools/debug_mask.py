import sys
sys.path.insert(0, '.')
import numpy as np, torch
import synth, oracle
import paper_1905_13038_b200 as ab
I = synth.page(512, 512, synth.config_seed(1))
ref = oracle.binarize("sauvola", I, 32, 32, 0.5, 128.0, stats=True)
x = torch.from_numpy(I).cuda()
m = ab.sauvola(x, 32, 32, 0.5, 128.0).cpu().numpy()
bad = np.argwhere(m != ref["mask"])
print("mismatches", len(bad), "got1", int(m.sum()), "want1", int(ref["mask"].sum()))
for (i, j) in bad[:10]:
    print(i, j, "I", I[i, j], "t", ref["t"][i, j], "c", ref["c"][i, j], "d", ref["d"][i, j], "n", ref["n"][i, j], "got", m[i, j])
# column pattern
if len(bad):
    print("cols mod 16", np.bincount(bad[:, 1] % 16, minlength=16))
    print("rows", np.unique(bad[:, 0])[:20])
