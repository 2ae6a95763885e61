import os, sys
sys.path.insert(0, '.')
import torch, synth
import paper_1905_13038_b200 as ab
P = torch.from_numpy(synth.pages(8, 4096, 4096, synth.config_seed(5))).cuda()
for _ in range(2): ab.binarize_batched("quantile", P, 51, 51, float(os.environ.get("Q", "0.5")))
torch.cuda.synchronize()
