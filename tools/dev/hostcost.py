"""Host cost per call (dev): the binding vs the raw C call vs torch helpers."""
import ctypes, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1905_13038_b200 as ab  # noqa: E402
from paper_1905_13038_b200 import abin  # noqa: E402

x = torch.zeros((512, 512), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
N = 100


def t(f, label):
    for _ in range(50):
        f()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(5e8))  # the GPU stays busy: the calls below only enqueue (no queue back-pressure)
    a = time.perf_counter()
    for _ in range(N):
        f()
    b = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{label:40s} {(b - a) / N * 1e6:7.2f} us/call")


t(lambda: ab.sauvola(x, 32, 32, 0.5, 128.0, out=out), "ab.sauvola")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
px, po = ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr())
t(lambda: abin._lib.abin_sauvola(px, 512, 512, 512, po, 512, 0, 32, 32, 0.5, 128.0, 0, None, st), "raw ctypes abin_sauvola")
t(lambda: torch.cuda.current_stream(), "torch.cuda.current_stream()")
t(lambda: (x.data_ptr(), x.stride(0), x.shape[0]), "tensor attrs")
os.environ["ABIN_SMALL_PX"] = "0"
t(lambda: abin._lib.abin_sauvola(px, 512, 512, 512, po, 512, 0, 32, 32, 0.5, 128.0, 0, None, st), "raw ctypes, streaming kernels")
