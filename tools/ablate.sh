#!/bin/bash
# Ablation builds of libsfseg_cuda.so (SFK_EXP bits: 1 = A arithmetic off,
# 2 = B arithmetic off) into /tmp/ablate/, for tools/time_solve.py.
set -e
cd "$(dirname "$0")/../paper_1907_02731_b200/csrc"
mkdir -p ../lib/ablate
for e in ${EXPS:-1 2 3}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       -diag-suppress 549 -DSFK_EXP=$e -shared -o ../lib/ablate/libsfseg_cuda_exp$e.so sfseg_api.cu &
done
wait
