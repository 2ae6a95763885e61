"""Build libabin.so (the CUDA kernels + C ABI) in-tree for sm_100a."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libabin.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-shared", "-Xptxas", "-warn-spills"]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))] + [
        os.path.join(ROOT, "include", "abin.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    newest = max(os.path.getmtime(s) for s in sources())
    if not force and not os.environ.get("ABIN_DEV_W32") and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    dev = os.environ.get("ABIN_DEV_W32")  # e.g. "29,5": development build, those w mod 32 classes only
    extra = []
    if dev:  # nvcc splits -D values at commas: pass the list through a header
        hdr = os.path.join(os.environ.get("TMPDIR", "/tmp"), "abin_dev_w32.h")
        with open(hdr, "w") as f:
            f.write("#define ABIN_DEV_W32 " + dev + "\n")
        extra = ["-include", hdr]
    cmd = [NVCC, *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp",
           os.path.join(CSRC, "abin_api.cu")]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
