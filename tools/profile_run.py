"""Small, fixed launch sequence of the bench workload, for ncu captures.

    python tools/profile_run.py [--kernel refill|naive] [--sims N] [--launches L] [--workload fixtures/c2_d1.json]

Runs L rollout launches (seeds 1..L) of every legal action x N sims through the
C-ABI on cuda:0 and prints the merged histogram checksum and the playouts per
launch (the divisor for per-playout ncu counters).
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="refill", choices=["refill", "naive"])
    ap.add_argument("--sims", type=int, default=1_000_000)
    ap.add_argument("--launches", type=int, default=2)
    ap.add_argument("--workload", default="fixtures/c2_d1.json")
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--grid", type=int, default=0)
    args = ap.parse_args()
    import torch
    from paper_2403_10720_b200 import dvc
    d = json.load(open(os.path.join(ROOT, args.workload)))
    st = dvc.encode(d)
    codes = st.legal_actions()
    dvc.set_option("kernel", {"refill": 0, "naive": 1}[args.kernel])
    if args.block:
        dvc.set_option("block", args.block)
    if args.grid:
        dvc.set_option("grid", args.grid)
    hist = torch.zeros((len(codes), st.players), dtype=torch.int64, device="cuda")
    for i in range(args.launches):
        dvc.rollout_batch_async(st, codes, 1 + i, 0, 0, args.sims, hist)
    torch.cuda.synchronize()
    print(json.dumps({"workload": args.workload, "kernel": args.kernel, "actions": len(codes),
                      "playouts_per_launch": len(codes) * args.sims, "launches": args.launches,
                      "hist_sum": int(hist.sum()), "n_det": st.info["n_det"]}))


if __name__ == "__main__":
    main()
