#!/bin/bash
# A/B of library builds on the multi-channel kernels (development aid):
# bit-identity against the first library and launch times on c4 / c2 crops.
# usage (GPU box): tools/ab_mc.sh base.so new.so ...
L="$@"
timeout 300 python tools/compare_libs.py --lib $L --config 4 --frames 64 --iters 4 --time || exit 1
timeout 300 python tools/compare_libs.py --lib $L --config 2 --iters 6 --time || exit 1
timeout 300 python tools/compare_libs.py --lib $L --config 4 --frames 12 --iters 3 --arith exact --time || exit 1
timeout 300 python tools/compare_libs.py --lib $L --config 2 --frames 12 --iters 6 --binarize 4 || exit 1
