#!/bin/bash
# A/B of the bench kernel time: current build vs paper_2403_10720_b200/libdvc_ab.so
# (DVC_LIB), alternating; prints kernel ms and playouts/s per run.  Extra
# arguments go to bench.py (e.g. --workload fixtures/c4_d1.json --sims 200000).
for i in 1 2 3; do
  for lib in libdvc_ab.so libdvc.so; do
    DVC_LIB=$lib python bench.py --no-cpu-baseline --steps 20 "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$lib', round(d['roofline']['kernel_ms'],4), '%.4g' % d['value'])"
  done
done
