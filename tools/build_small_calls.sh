#!/bin/bash
# builds build/small_calls against the drop-in (needs /root/reference headers)
set -e
cd "$(dirname "$0")/.."
mkdir -p build
g++ -std=c++20 -O2 -I/root/reference/proj/include -o build/small_calls tools/small_calls.cpp \
  -Lpaper_1907_02731_b200/lib -lsfseg_engine_cuda -lsfseg_cuda oracle/_ref/libsfseg_ref_noengine.a \
  -Wl,-rpath,'$ORIGIN/../paper_1907_02731_b200/lib' -lpthread
echo built build/small_calls
