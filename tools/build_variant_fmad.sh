#!/bin/bash
# usage: tools/build_variant.sh NAME [extra nvcc flags...] -- build libsimplets.so variant into build/NAME.so (A/B experiments)
N=$1; shift
cd "$(dirname "$0")/../paper_1802_04243_b200/csrc" && \
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
   -Xptxas -v "$@" -o ../../build/$N.so simplets.cu > ../../build/$N.ptxas.log 2>&1 && \
grep -A2 "march_kernelILb" ../../build/$N.ptxas.log | grep -E "spill|Used" | paste - - | awk '{print $5,$6,$7,$8,$16,$17}'
