#!/bin/bash
# Build an A/B variant of libdvc.so: tools/build_ab.sh OUT.so [nvcc -D flags ...]
# e.g. tools/build_ab.sh libdvc_ab.so -DDVC_REFILL_MINB=4 ; then tools/ab_bench.sh
OUT=$1; shift
H=paper_2403_10720_b200
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -shared \
  -Xcompiler -fPIC -Xcompiler -O2 -Xcompiler -ffp-contract=off -I include "$@" -o $H/$OUT \
  $H/csrc/api.cu $H/csrc/kernels.cu $H/csrc/host.cpp $H/csrc/mcts.cpp
