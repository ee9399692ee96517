#!/bin/bash
# Development aid: build libsfseg_cuda.so with extra -D flags into
# build/exp/NAME/ (travels to the GPU box; compare with tools/time_solve.py --lib ...)
# usage: tools/build_variant.sh NAME [-DSFK_...=v ...]
set -e
NAME=$1; shift
OUT=build/exp/$NAME
mkdir -p "$OUT"
cd paper_1907_02731_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -diag-suppress 549,177 "$@" -shared -o "../../$OUT/libsfseg_cuda.so" sfseg_api.cu synth_dev.cu
echo "built $OUT"
