#!/bin/bash
# One gpurun call that regenerates every number profiles/ holds for a round:
#   tools/round_measure.sh TAG   (outputs under gpurun_out/TAG/)
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
set -x
python tools/configs_bench.py > $O/configs.jsonl 2> $O/configs.err
python tools/c5_sweep.py --out $O --tag $TAG > $O/c5.log 2>&1
python tools/paper_experiments.py --out $O --tag $TAG > $O/exp.log 2>&1
python tools/search_latency.py > $O/${TAG}_search_latency_c3.jsonl 2> $O/sl.err
python tools/search_latency_deep.py > $O/${TAG}_search_latency_deep.jsonl 2> $O/sld.err
# launch list of the bench command (cold-cache, serialised; compare shares)
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c4 --no-deals > $O/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ncu.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c4 --no-deals > $O/ncu_launch.log 2>&1
# full captures of the dominant kernels
python tools/profile_run.py --launches 2 > $O/p1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rollout_refill -s 1 -c 1 -o $O/refill_c2 \
      python tools/profile_run.py --launches 2 > /dev/null 2>&1
python tools/profile_run.py --launches 2 --kernel naive --block 1024 > $O/p2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rollout_naive -s 1 -c 1 -o $O/naive_c2 \
      python tools/profile_run.py --launches 2 --kernel naive --block 1024 > /dev/null 2>&1
python tools/profile_run.py --launches 2 --workload fixtures/c4_d1.json --sims 100000 > $O/p3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rollout_refill -s 1 -c 1 -o $O/refill_c4 \
      python tools/profile_run.py --launches 2 --workload fixtures/c4_d1.json --sims 100000 > /dev/null 2>&1
# the bench line last, with the per-playout instruction count of the capture above
python tools/summarize_profile.py $O/refill_c2.ncu-rep 21000000 $O/refill_c2_summary.json --unit > /dev/null
python bench.py > $O/bench.jsonl 2> $O/bench.err
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipes tools/micro/pipes.cu && /tmp/pipes > $O/${TAG}_pipes.txt 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.jsonl 2> $O/bench_ref.err
echo done
