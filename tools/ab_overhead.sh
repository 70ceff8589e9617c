#!/bin/bash
# A/B of the per-call overhead (tools/overhead.py) between the current build
# and another build copied to paper_2403_10720_b200/libdvc_ab.so (selected by
# DVC_LIB), alternating three times on the same box.
for i in 1 2 3; do
DVC_LIB=libdvc_ab.so python tools/overhead.py | sed 's/^/OLD /'
python tools/overhead.py | sed 's/^/NEW /'
done
