"""Launch-configuration sweep (the C5 / N2 harness, PAPER:222-257 figures
`fig:gpu_num_simulation`, `fig:gpu_warp_simulation`, `fig:gpu_thread_time`):
playouts/s of both kernels over block x grid on one workload, with the
histogram checked identical at every point (results never depend on the
launch configuration).

    python tools/sweep.py [--workload fixtures/c2_d1.json] [--sims N] [--blocks 32,64,...]
                          [--grids 0,1,...] [--kernels refill,naive] [--reps 3] [--csv out.csv]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="fixtures/c2_d1.json")
    ap.add_argument("--sims", type=int, default=1_000_000)
    ap.add_argument("--blocks", default="64,128,256,512")
    ap.add_argument("--grids", default="0")
    ap.add_argument("--kernels", default="refill,naive")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--csv", default=None)
    args = ap.parse_args()
    import torch
    from paper_2403_10720_b200 import dvc
    d = json.load(open(os.path.join(ROOT, args.workload)))
    st = dvc.encode(d)
    codes = st.legal_actions()
    A, P = len(codes), st.players
    hist = torch.zeros((A, P), dtype=torch.int64, device="cuda")
    ref = None
    rows = []
    stream = torch.cuda.current_stream()
    for kern in args.kernels.split(","):
        for blk in [int(x) for x in args.blocks.split(",")]:
            for grid in [int(x) for x in args.grids.split(",")]:
                with dvc.options(kernel=1 if kern == "naive" else 0, block=blk, grid=grid):
                    hist.zero_()
                    dvc.rollout_batch_async(st, codes, 1, 0, 0, args.sims, hist)   # warm-up + check
                    torch.cuda.synchronize()
                    h = hist.cpu()
                    if ref is None:
                        ref = h
                    ok = bool(torch.equal(h, ref))
                    best = None
                    for r in range(args.reps):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        dvc.rollout_batch_async(st, codes, 1, 0, 0, args.sims, hist)
                        e1.record(stream)
                        torch.cuda.synchronize()
                        ms = e0.elapsed_time(e1)
                        best = ms if best is None else min(best, ms)
                    pps = A * args.sims / (best / 1000.0)
                    row = {"kernel": kern, "block": blk, "grid": grid, "ms": round(best, 4),
                           "playouts_per_s": pps, "hist_identical": ok}
                    rows.append(row)
                    print(json.dumps(row), flush=True)
    if args.csv:
        with open(args.csv, "w") as f:
            f.write("kernel,block,grid,ms,playouts_per_s,hist_identical\n")
            for r in rows:
                f.write("%s,%d,%d,%.4f,%.6e,%d\n" % (r["kernel"], r["block"], r["grid"], r["ms"],
                                                    r["playouts_per_s"], r["hist_identical"]))


if __name__ == "__main__":
    main()
