"""C5: the paper's launch-configuration sweeps on one B200 (SURVEY §8(d) C5,
§8(f) N2), for both kernels, on the C2 fixture (deal 1, consecutive rules).

  * threads (fig:gpu_num_simulation; fig:gpu_thread_time,
    PAPER:245-257): ONE block of T threads, T = 1..1024, weak scaling at
    `--per-thread` playouts per thread: kernel time and playouts/s;
  * warps (fig:gpu_warp_simulation): one block of 1..32 warps;
  * device: blocks x threads over the whole GPU at a fixed 2^24 playouts
    (strong scaling), including the auto (persistent) configuration.

Every point's winner histogram is compared with the first point of the same
workload (results never depend on the launch configuration).
Writes CSVs under --out (default profiles/) with SPEC:370's columns extended.

    python tools/c5_sweep.py [--out profiles] [--per-thread 64] [--tag r01]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--per-thread", type=int, default=64)
    ap.add_argument("--device-playouts", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from paper_2403_10720_b200 import dvc
    d = json.load(open(os.path.join(ROOT, "fixtures", "c2_d1.json")))
    st = dvc.encode(d)
    codes = st.legal_actions()
    A, P = len(codes), st.players
    stream = torch.cuda.current_stream()
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    hist = torch.zeros((A, P), dtype=torch.int64, device="cuda")

    def run(kernel, block, grid, total):
        """total playouts spread over all actions -> (best ms, hist)."""
        n = max(1, total // A)
        best = None
        h = None
        with dvc.options(kernel=kernel, block=block, grid=grid):
            for r in range(args.reps + 1):
                hist.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                dvc.rollout_batch_async(st, codes, 1, 0, 0, n, hist)
                e1.record(stream)
                torch.cuda.synchronize()
                if r == 0:
                    h = hist.cpu()
                    continue                      # warm-up
                ms = e0.elapsed_time(e1)
                best = ms if best is None else min(best, ms)
        return best, h, n * A

    os.makedirs(args.out, exist_ok=True)
    hdr = "run,workers,total_simulations,elapsed_ns,sims_per_sec,device,gpus,block,grid,kernel,hist_identical\n"

    # --- one block, T threads (naive: any T; refill: whole warps), weak scaling
    refs = {}
    rows = []
    for T in [1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 160, 192, 224, 256, 320, 384, 448, 512, 640, 768, 896, 1024]:
        for kern, kname in ((1, "naive"), (0, "refill")):
            if kern == 0 and (T % 32 or T > 256):
                continue
            total = T * args.per_thread
            ms, h, done = run(kern, T, 1, total)
            key = done
            same = None
            if key in refs:
                same = bool(torch.equal(refs[key], h))
            else:
                refs[key] = h
            rows.append((-1, T, done, int(ms * 1e6), done / (ms / 1e3), "B200", 1, T, 1, kname, same))
            print(json.dumps({"sweep": "threads", "kernel": kname, "threads": T, "playouts": done, "ms": ms,
                              "playouts_per_s": done / (ms / 1e3), "hist_identical": same}), flush=True)
    with open(os.path.join(args.out, "%s_c5_threads.csv" % args.tag), "w") as f:
        f.write(hdr)
        for r in rows:
            f.write("%d,%d,%d,%d,%.6e,%s,%d,%d,%d,%s,%s\n" % r)

    # --- full device, fixed work (strong scaling)
    rows = []
    ref = None
    total = args.device_playouts
    grids = [1, 2, 8, 37, 74, 148, 296, 592, 1184, 0]
    for kern, kname, blocks in ((1, "naive", [32, 64, 128, 256, 512, 1024]), (0, "refill", [32, 64, 128, 256])):
        for blk in blocks:
            for g in grids:
                if g and g * blk < 32 * 64:
                    continue                     # too small to finish 2^24 playouts in reasonable time
                ms, h, done = run(kern, blk, g, total)
                if ref is None:
                    ref = h
                same = bool(torch.equal(ref, h))
                rows.append((-1, blk * (g or 0), done, int(ms * 1e6), done / (ms / 1e3), "B200", 1, blk, g, kname,
                             same))
                print(json.dumps({"sweep": "device", "kernel": kname, "block": blk, "grid": g or "auto",
                                  "ms": ms, "playouts_per_s": done / (ms / 1e3), "hist_identical": same}),
                      flush=True)
    with open(os.path.join(args.out, "%s_c5_device.csv" % args.tag), "w") as f:
        f.write(hdr.replace("workers", "threads_total"))
        for r in rows:
            f.write("%d,%d,%d,%d,%.6e,%s,%d,%d,%d,%s,%s\n" % r)
    print(json.dumps({"sm_count": n_sm, "actions": A}))


if __name__ == "__main__":
    main()
