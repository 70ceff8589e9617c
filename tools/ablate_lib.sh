#!/bin/bash
# Time the C2 workload with alternative builds of libdvc.so (ablation of
# compile-time knobs): tools/ablate_lib.sh lib1.so lib2.so ...
for L in "$@"; do
  cp "$L" paper_2403_10720_b200/libdvc.so
  echo "== $L"
  python tools/sweep.py --blocks 64,128 --kernels refill --reps 5 2>&1 | tail -2
done
