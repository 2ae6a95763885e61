"""Build libabin.so (the CUDA kernels + C ABI) in-tree for sm_100a.

The kernel template instantiations are spread over several translation units
(csrc/moments_part.cu x 8, csrc/wide_part.cu x 2, csrc/quant5_part.cu x 4,
csrc/abin_api.cu) that nvcc
compiles in parallel into build/*.o; they are then linked into one shared
library.
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libabin.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"]
N_PARTS = 8


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))] + [
        os.path.join(ROOT, "include", "abin.h")]


def units():
    """(object name, source, extra flags) for every translation unit."""
    u = [("abin_api.o", "abin_api.cu", [])]
    u += [(f"moments_part{k}.o", "moments_part.cu", [f"-DABIN_PART={k}"]) for k in range(N_PARTS)]
    u += [(f"wide_part{d}.o", "wide_part.cu", [f"-DABIN_WIDE_D64={d}"]) for d in (0, 1)]
    u += [(f"quant5_part{k}.o", "quant5_part.cu", [f"-DABIN_Q5_PART={k}"]) for k in range(4)]
    return u


def build(force: bool = False, verbose: bool = False, extra=(), lib: str = LIB, obj: str = OBJ) -> str:
    """Compile every unit and link `lib`.  `extra` (nvcc flags) and another
    `lib` / `obj` are for development A/B builds (tools/abbuild.py)."""
    newest = max(os.path.getmtime(s) for s in sources() + [os.path.abspath(__file__)])
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= newest:
        return lib
    os.makedirs(obj, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")]

    obj_dir = obj

    def compile_one(unit):
        o, src, extra_u = unit
        cmd = [NVCC, *NVCC_FLAGS, *extra_u, *extra, *inc, "-c", "-o", os.path.join(obj_dir, o), os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src} {extra}:\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, file=sys.stderr)
        return o

    with ThreadPoolExecutor(max_workers=max(1, min(len(units()), os.cpu_count() or 4))) as ex:
        objs = list(ex.map(compile_one, units()))
    cmd = [NVCC, *ARCH, "-shared", "-o", lib + ".tmp", *[os.path.join(obj_dir, o) for o in objs]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
