"""Development A/B builds of libabin.so with extra nvcc flags, e.g.
    python tools/abbuild.py minb18 -DABIN_V5_MINB=18
writes paper_1905_13038_b200/ab/libabin_<tag>.so; load it with ABIN_LIB=<path>."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_1905_13038_b200"))
import build  # noqa: E402

tag, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "paper_1905_13038_b200", "ab")
os.makedirs(out, exist_ok=True)
print(build.build(force=True, extra=flags, lib=os.path.join(out, f"libabin_{tag}.so"),
                  obj=os.path.join(out, f"obj_{tag}")))
