#!/bin/bash
# Variant builds of libsfseg_cuda.so for kernel experiments:
#   tools/ablate_mc.sh "name:-DFLAG=1 -DOTHER=2" ...
#     -> paper_1907_02731_b200/lib/exp/libsfseg_cuda_<name>.so (time with tools/time_solve.py --lib)
set -e
cd "$(dirname "$0")/../paper_1907_02731_b200/csrc"
mkdir -p ../lib/exp
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       -diag-suppress 549 $flags -shared -o ../lib/exp/libsfseg_cuda_$name.so sfseg_api.cu &
done
wait
ls -la ../lib/exp
