#!/bin/bash
# Build a variant of libchap.so into vlibs/NAME.so with extra nvcc flags (experiments only).
#   tools/vbuild.sh NAME [-DFOO ...]
set -e
N=$1; shift
mkdir -p vlibs
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 -shared \
  --expt-relaxed-constexpr -Iinclude -Ipaper_2605_05086_b200/csrc "$@" -o vlibs/$N.so paper_2605_05086_b200/csrc/chap.cu -ldl
