#!/bin/bash
# tools/abbuild.sh <name> <extra nvcc flags...>: build a variant libabin into abvar/<name>.so (for A/B timing)
name=$1; shift
mkdir -p abvar/$name.obj
cd paper_1905_13038_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include"
pids=()
/usr/local/cuda/bin/nvcc $F "$@" -c -o ../../abvar/$name.obj/api.o abin_api.cu & pids+=($!)
for k in 0 1 2 3 4 5 6 7; do /usr/local/cuda/bin/nvcc $F "$@" -DABIN_PART=$k -c -o ../../abvar/$name.obj/p$k.o moments_part.cu & pids+=($!); done
for d in 0 1; do /usr/local/cuda/bin/nvcc $F "$@" -DABIN_WIDE_D64=$d -c -o ../../abvar/$name.obj/w$d.o wide_part.cu & pids+=($!); done
for p in ${pids[@]}; do wait $p || exit 1; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../abvar/$name.so ../../abvar/$name.obj/*.o
rm -rf ../../abvar/$name.obj
echo built abvar/$name.so
