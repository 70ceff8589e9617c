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


def cpu_rows(exp, steps, sizes=None):
    """The CPU (oracle) side runs in bench.py's reference arm (the only place
    besides tests/ allowed to execute oracle/); returns its rows."""
    import subprocess
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--ref-sweep", exp,
           "--steps", str(steps)]
    if sizes:
        cmd += ["--ref-sizes", ",".join(map(str, sizes))]
    out = subprocess.run(cmd, capture_output=True, text=True, check=True, cwd=ROOT).stdout
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--cpu-max", type=int, default=1_000_000)
    ap.add_argument("--repeats", type=int, default=5)
    args = ap.parse_args()
    import torch
    from paper_2403_10720_b200 import dvc
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
    for r in cpu_rows("exp1", args.repeats, [n for n in sizes if n <= args.cpu_max]):
        rows.append((r["run"], r["workers"], r["total_simulations"], r["elapsed_ns"], r["sims_per_sec"], "cpu",
                     "oracle"))
    with open(os.path.join(args.out, "%s_exp1_time_vs_sims.csv" % args.tag), "w") as f:
        f.write(hdr)
        for r in rows:
            f.write("%d,%d,%d,%d,%.6e,%s,%s\n" % r)

    # ---- EXP-2: CPU sims/s vs workers (bench.py reference arm)
    rows = [(r["run"], r["workers"], r["total_simulations"], r["elapsed_ns"], r["sims_per_sec"], "cpu", "oracle")
            for r in cpu_rows("exp2", 3)]
    with open(os.path.join(args.out, "%s_exp2_cpu_workers.csv" % args.tag), "w") as f:
        f.write(hdr)
        for r in rows:
            f.write("%d,%d,%d,%d,%.6e,%s,%s\n" % r)
    # ---- the oracle on one pinned core, first 10^6 playouts of C2
    one = cpu_rows("core1", 1)
    with open(os.path.join(args.out, "%s_cpu_1core.json" % args.tag), "w") as f:
        json.dump(one[-1] if one else None, f, indent=1)
    print(json.dumps({"cores": cores, "one_core": one[-1] if one else None}))


if __name__ == "__main__":
    main()
