import os, sys
sys.path.insert(0, '.')
import numpy as np, torch, synth, oracle
import paper_1905_13038_b200 as ab
from paper_1905_13038_b200 import abin
os.environ["ABIN_HOSTIO_CHUNK_BYTES"] = "20000"
P, H, W = 3, 230, 333
pages = synth.pages(P, H, W, synth.config_seed(3), stain=True)
pages[1, 100:140] = 200
for method, p0 in (("bernsen", 15.0), ("quantile", 0.5)):
    hin = torch.from_numpy(pages).pin_memory()
    hout = torch.zeros((P, H, W), dtype=torch.uint8).pin_memory()
    rc = abin.raw().abin_binarize_batched(abin.METHODS[method], abin.ctypes.c_void_p(hin.data_ptr()), hin.stride(0),
        abin.ctypes.c_void_p(hout.data_ptr()), hout.stride(0), P, H, W, hin.stride(1), hout.stride(1), abin.MASK_U8, 31, 25,
        p0, 0.0, -1, abin.HOST_IO, None, abin.ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    got = hout.numpy()
    for p in range(P):
        ref = oracle.bernsen(pages[p], 31, 25, 15)[0] if method == "bernsen" else oracle.quantile(pages[p], 31, 25, 0.5)[0]
        d = np.nonzero(got[p] != ref)
        print(method, rc, p, "mismatches", d[0].size, "rows", np.unique(d[0])[:12], "cols", np.unique(d[1])[:12])
