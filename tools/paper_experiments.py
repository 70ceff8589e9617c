"""The paper's CPU/GPU experiments re-run on this build:

  EXP-1 (fig:time_consuming): execution time vs number of
        simulations (1 .. 10^7), mean of 5 runs, on the GPU (refill kernel,
        whole device) and the CPU oracle (all host cores);
  EXP-2 (fig:cpu_num_simulation): CPU simulations/s vs worker
        processes 1 .. 2x cores (the oracle, one process per worker).

Workload: the C2 fixture (deal 1), simulations spread over its legal actions.
CSV columns follow SPEC:370 (run,workers,total_simulations,elapsed_ns,
sims_per_sec) with device/kernel appended; run = -1 rows are the means.

    python tools/paper_experiments.py [--out profiles] [--tag r01] [--cpu-max 1000000]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _job(args):
    import oracle
    d, codes, seed, s0, s1 = args
    return oracle.rollout(d, codes, seed, 0, s0, s1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--cpu-max", type=int, default=1_000_000)
    ap.add_argument("--repeats", type=int, default=5)
    args = ap.parse_args()
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    import torch
    import oracle
    from paper_2403_10720_b200 import dvc
    oracle.build()
    d = json.load(open(os.path.join(ROOT, "fixtures", "c2_d1.json")))
    st = dvc.encode(d)
    codes = st.legal_actions()
    A = len(codes)
    cores = os.cpu_count() or 1
    os.makedirs(args.out, exist_ok=True)
    hdr = "run,workers,total_simulations,elapsed_ns,sims_per_sec,device,kernel\n"

    # ---- EXP-1: time vs simulations
    rows = []
    sizes = [1, 10, 100, 1000, 10 ** 4, 10 ** 5, 10 ** 6, 10 ** 7]
    hist = torch.zeros((A, st.players), dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    pool = ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("spawn"))
    list(pool.map(_job, [(d, codes, 1, 0, 1)] * cores))                  # warm the workers
    for n in sizes:
        # GPU: n simulations over the actions (the first n mod A actions get one more)
        per, extra = divmod(n, A)
        acts_full, acts_extra = codes, codes[:extra]
        ts = []
        for r in range(args.repeats + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            hist.zero_()
            e0.record(stream)
            if per:
                dvc.rollout_batch_async(st, acts_full, 1 + r, 0, 0, per, hist)
            if extra:
                dvc.rollout_batch_async(st, acts_extra, 1 + r, 0, per, per + 1, hist[:extra])
            e1.record(stream)
            torch.cuda.synchronize()
            assert int(hist.sum()) == n
            if r:
                ts.append(e0.elapsed_time(e1) * 1e6)
        for i, t in enumerate(ts):
            rows.append((i, 1, n, int(t), n / (t / 1e9), "B200", "refill"))
        rows.append((-1, 1, n, int(sum(ts) / len(ts)), n / (sum(ts) / len(ts) / 1e9), "B200", "refill"))
        print(json.dumps({"exp": 1, "device": "gpu", "sims": n, "mean_ms": sum(ts) / len(ts) / 1e6}), flush=True)
        if n <= args.cpu_max:
            ts = []
            for r in range(args.repeats):
                jobs = []
                for w in range(cores):
                    a0, a1 = (per * w) // cores, (per * (w + 1)) // cores
                    if a1 > a0:
                        jobs.append((d, codes, 1 + r, a0, a1))
                if extra:
                    jobs.append((d, codes[:extra], 1 + r, per, per + 1))
                t0 = time.perf_counter()
                list(pool.map(_job, jobs))
                ts.append((time.perf_counter() - t0) * 1e9)
            for i, t in enumerate(ts):
                rows.append((i, cores, n, int(t), n / (t / 1e9), "cpu", "oracle"))
            rows.append((-1, cores, n, int(sum(ts) / len(ts)), n / (sum(ts) / len(ts) / 1e9), "cpu", "oracle"))
            print(json.dumps({"exp": 1, "device": "cpu", "workers": cores, "sims": n,
                              "mean_ms": sum(ts) / len(ts) / 1e6}), flush=True)
    pool.shutdown()
    with open(os.path.join(args.out, "%s_exp1_time_vs_sims.csv" % args.tag), "w") as f:
        f.write(hdr)
        for r in rows:
            f.write("%d,%d,%d,%d,%.6e,%s,%s\n" % r)

    # ---- EXP-2: CPU sims/s vs workers
    rows = []
    n_per_worker = 4000
    for w in sorted({1, 2, 4, 8, 12, 16, 24, 32, cores, 2 * cores}):
        if w > 2 * cores:
            continue
        with ProcessPoolExecutor(max_workers=w, mp_context=mp.get_context("spawn")) as ex:
            list(ex.map(_job, [(d, codes[:1], 1, 0, 1)] * w))
            ts = []
            for r in range(3):
                jobs = [(d, codes[:4], 1 + r, i * n_per_worker, (i + 1) * n_per_worker) for i in range(w)]
                t0 = time.perf_counter()
                list(ex.map(_job, jobs))
                ts.append(time.perf_counter() - t0)
            total = w * n_per_worker * 4
            for i, t in enumerate(ts):
                rows.append((i, w, total, int(t * 1e9), total / t, "cpu", "oracle"))
            m = sum(ts) / len(ts)
            rows.append((-1, w, total, int(m * 1e9), total / m, "cpu", "oracle"))
            print(json.dumps({"exp": 2, "workers": w, "sims_per_s": total / m}), flush=True)
    with open(os.path.join(args.out, "%s_exp2_cpu_workers.csv" % args.tag), "w") as f:
        f.write(hdr)
        for r in rows:
            f.write("%d,%d,%d,%d,%.6e,%s,%s\n" % r)
    print(json.dumps({"cores": cores}))


if __name__ == "__main__":
    main()
