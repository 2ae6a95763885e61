import os, sys
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
I = synth.page(4096, 4096, synth.config_seed(5))
x = torch.from_numpy(I).cuda()
q = float(os.environ.get("Q", "0.5"))
for _ in range(3): ab.binarize_batched("quantile", x.unsqueeze(0), 51, 51, q)
torch.cuda.synchronize()
