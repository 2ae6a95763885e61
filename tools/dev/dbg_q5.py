import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch, synth, oracle
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin
from test_gpu_quant5 import run
I = synth.page(90, 700, synth.config_seed(5, 11))
for fl in (None, "0", "240", "100"):
    if fl is None: os.environ.pop("ABIN_Q5_FORCE_L", None)
    else: os.environ["ABIN_Q5_FORCE_L"] = fl
    for q, packed in ((0.5, False), (0.1, True), (0.5, True), (0.1, False)):
        got, n = run(I, 21, 33, q, packed)
        ref = oracle.quantile(I, 21, 33, q)[0]
        want = oracle.pack_bits(ref) if packed else ref
        print(fl, q, packed, 'n_exact', n, 'match', np.array_equal(got, want), flush=True)
