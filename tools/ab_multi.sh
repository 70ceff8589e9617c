#!/bin/bash
# A/B/n of the bench kernel time over several builds, interleaved:
#   tools/ab_multi.sh "libA.so libB.so ..." [bench.py args]
LIBS=$1; shift
for i in 1 2 3; do
  for lib in $LIBS; do
    DVC_LIB=$lib python bench.py --no-cpu-baseline --steps 20 "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$lib', round(d['roofline']['kernel_ms'],4), '%.4g' % d['value'])"
  done
done
