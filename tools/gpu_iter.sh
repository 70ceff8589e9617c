#!/bin/bash
# One build->measure iteration on the GPU box (run under gpurun):
#   parity subset, bench both kernels, ncu --set full of both kernels.
# usage: tools/gpu_iter.sh TAG [pytest -k expr]
TAG=${1:-iter}
K=${2:-"golden or schedule or edge or async or full_size or c2_d1 or c4_d2 or x3_d1"}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $O/tests.log 2>&1; echo "tests=$?"; tail -3 $O/tests.log
for kern in refill naive; do
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --kernel $kern > $O/bench_$kern.log 2>&1 || echo "bench $kern failed"
  python - $O/bench_$kern.log <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d=json.loads(l); print(d["config"]["kernel"], "%.3e playouts/s" % d["value"], "kernel_ms %.3f" % d["roofline"]["kernel_ms"], "e2e %.3e" % d["e2e"]["value"], d["clocks"])
PY
done
python tools/profile_run.py --launches 2 > $O/plain_refill.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rollout_refill -s 1 -c 1 -o $O/refill python tools/profile_run.py --launches 2 > $O/ncu_refill.log 2>&1; echo "ncu_refill=$?"
python tools/profile_run.py --launches 2 --kernel naive > $O/plain_naive.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rollout_naive -s 1 -c 1 -o $O/naive python tools/profile_run.py --launches 2 --kernel naive > $O/ncu_naive.log 2>&1; echo "ncu_naive=$?"
