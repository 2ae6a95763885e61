#!/bin/bash
# A/B of the quantile kernel builds: config 5 page and 8-page batch
for lib in paper_1905_13038_b200/libabin.so paper_1905_13038_b200/ab/libabin_mb14.so paper_1905_13038_b200/ab/libabin_mb16.so; do
  echo "== $lib"
  ABIN_LIB=$lib timeout 300 python tools/dev/q5_sweep.py 2>&1 | grep -E "default q=0.5|5b"
done
