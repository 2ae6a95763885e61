import sys, os, time
sys.path.insert(0, '.')
import numpy as np, torch, synth
from paper_1905_13038_b200 import abin
P, H, W = 64, 7016, 4960
pages = synth.pages(P, H, W, synth.config_seed(3), stain=True)
hin = torch.from_numpy(pages).pin_memory(); hout = torch.empty((P, H, W), dtype=torch.uint8).pin_memory()
cs = torch.cuda.current_stream()
def step():
    rc = abin.raw().abin_binarize_batched(0, abin.ctypes.c_void_p(hin.data_ptr()), hin.stride(0), abin.ctypes.c_void_p(hout.data_ptr()), hout.stride(0), P, H, W, W, W, 0, 61, 61, 0.5, 128.0, -1, abin.HOST_IO, None, abin.ctypes.c_void_p(cs.cuda_stream))
    assert rc == 0
step(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); [step() for _ in range(3)]; b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
print(os.environ.get("ABIN_HOSTIO_CHUNK_MB"), os.environ.get("ABIN_HOSTIO_STREAMS"), f"{ms:.1f} ms {P*H*W/ms/1e6:.1f} Gpx/s")
