#!/bin/bash
# A/B of library builds on the register-ring FAST kernels (development aid):
# bit-identity against the first library on c0, a c1 crop with binarised
# iterations, a c3 clip, then launch times at full c1 and on a c3 clip.
# usage (GPU box): tools/ab_rs.sh build/exp/base/libsfseg_cuda.so build/exp/new/libsfseg_cuda.so ...
L="$@"
python tools/compare_libs.py --lib $L --config 0 || exit 1
python tools/compare_libs.py --lib $L --config 1 --frames 20 --iters 8 --binarize 5 || exit 1
python tools/compare_libs.py --lib $L --config 3 --clip 2 --frames 40 --iters 6 --time || exit 1
python tools/compare_libs.py --lib $L --config 1 --time || exit 1
