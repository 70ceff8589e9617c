"""Per-config measurements of BASELINE.json configs C1-C4 (SURVEY §8(d)
table) on one B200, each checked for internal consistency (every playout
accounted for).  Prints one JSON line per config.

    python tools/configs_bench.py [--configs c1,c2,c3,c4] [--reps 5]

C1: latency of one decision (encode + dvc_rollout_batch: H2D, kernels, D2H),
    all legal actions x 1000 playouts, 8 opening deals.
C2: kernel throughput at 10^6 playouts per action, 8 mid-game deals.
C3: full self-play games (2p, 26 tiles with jokers), each decision a
    dvc_mcts_search (64 expansions x 1024 sims per child; flat and
    depth-capped): decisions/s.
C4: 4 players, 26 tiles, 3 each: ceil(1e8 / A) playouts per action (~1e8 per
    move) on one GPU, 8 deals: playouts/s (the 8-GPU run is bench.py's job).
"""

import argparse
import glob
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    from paper_2403_10720_b200 import dvc
    stream = torch.cuda.current_stream()
    todo = args.configs.split(",")

    def load(pat):
        return [json.load(open(p)) for p in sorted(glob.glob(os.path.join(ROOT, "fixtures", pat)))]

    def kernel_time(st, codes, n, seed):
        hist = torch.zeros((len(codes), st.players), dtype=torch.int64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dvc.rollout_batch_async(st, codes, seed, 0, 0, n, hist)
        e1.record(stream)
        torch.cuda.synchronize()
        assert int(hist.sum()) == n * len(codes)
        return e0.elapsed_time(e1) / 1000.0

    if "c1" in todo:
        lat, pps = [], []
        for d in load("c1_d*.json"):
            st = dvc.encode(d)
            codes = st.legal_actions()
            dvc.rollout_batch(st, codes, 1000, 99)          # warm
            ts = []
            for r in range(args.reps):
                t0 = time.perf_counter()
                st2 = dvc.encode(d)
                w = dvc.rollout_batch(st2, codes, 1000, 1 + r)
                ts.append(time.perf_counter() - t0)
            t = min(ts)
            lat.append(t)
            pps.append(1000 * len(codes) / t)
        print(json.dumps({"config": "C1", "desc": "2p/24 tiles/opening, all legal x 1000, per decision",
                          "latency_ms_min_per_deal": [round(1e3 * x, 3) for x in lat],
                          "latency_ms_mean": 1e3 * sum(lat) / len(lat),
                          "playouts_per_s_mean": sum(pps) / len(pps)}), flush=True)
    if "c2" in todo:
        rows = []
        for i, d in enumerate(load("c2_d*.json")):
            st = dvc.encode(d)
            codes = st.legal_actions()
            kernel_time(st, codes, 1000000, 77)
            t = min(kernel_time(st, codes, 1000000, 1 + r) for r in range(args.reps))
            rows.append({"deal": i + 1, "actions": len(codes), "ms": round(1e3 * t, 3),
                         "playouts_per_s": len(codes) * 1e6 / t})
        print(json.dumps({"config": "C2", "desc": "2p/24 tiles/mid-game, all legal x 1e6", "per_deal": rows,
                          "playouts_per_s_mean": sum(r["playouts_per_s"] for r in rows) / len(rows)}), flush=True)
    if "c3" in todo:
        # full self-play games (2p, 26 tiles with jokers), every decision a
        # dvc_mcts_search of 64 expansions x 1024 playouts per child
        from paper_2403_10720_b200.selfplay import play_game
        for flat, sdev, label in ((1, 1, "flat UCT (root-parallel, PAPER:180), device-resident UCB loop"),
                                  (1, 0, "flat UCT (root-parallel, PAPER:180), host UCB loop"),
                                  (0, 0, "depth-capped tree, max_depth 4, host tree"),
                                  (0, 1, "depth-capped tree, max_depth 4, device-resident tree")):
            dvc.set_option("search_device", sdev)
            rows = []
            dvc.mcts_search(dvc.encode(load("c3_d*.json")[0]), 4, 1024, 5, flat=flat)
            for g in range(4):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = play_game(100 + g, expansions=64, sims_per_child=1024, flat=flat, max_depth=4)
                t = time.perf_counter() - t0
                rows.append({"game": 100 + g, "decisions": res["decisions"], "winner": res["winner"],
                             "s": round(t, 3), "ms_per_decision": round(1e3 * t / res["decisions"], 3)})
            dec = sum(r["decisions"] for r in rows)
            tt = sum(r["s"] for r in rows)
            # the same kind of games, 16 at a time on 16 host threads / CUDA streams
            from paper_2403_10720_b200.selfplay import play_games
            t0 = time.perf_counter()
            many = play_games(list(range(200, 216)), threads=16, expansions=64, sims_per_child=1024, flat=flat,
                              max_depth=4)
            tm = time.perf_counter() - t0
            print(json.dumps({"config": "C3", "desc": "2p/26 tiles (jokers) self-play games, %s, 64 x 1024 per "
                              "decision" % label, "games": rows, "decisions_per_s": dec / tt,
                              "concurrent_16_games": {"decisions": sum(g["decisions"] for g in many), "s": round(tm, 3),
                                                      "decisions_per_s": sum(g["decisions"] for g in many) / tm}}),
                  flush=True)
        dvc.set_option("search_device", 0)
    if "c4" in todo:
        rows = []
        for i, d in enumerate(load("c4_d*.json")):
            st = dvc.encode(d)
            codes = st.legal_actions()
            n = -(-100000000 // len(codes))
            kernel_time(st, codes, 10000, 77)               # builds the det table
            t = min(kernel_time(st, codes, n, 1 + r) for r in range(max(1, args.reps // 2)))
            rows.append({"deal": i + 1, "actions": len(codes), "n_det": st.info["n_det"], "sims_per_action": n,
                         "ms": round(1e3 * t, 2), "playouts_per_s": len(codes) * n / t})
        print(json.dumps({"config": "C4", "desc": "4p/26 tiles/3 each, ~1e8 playouts per move, 1 GPU",
                          "per_deal": rows,
                          "playouts_per_s_mean": sum(r["playouts_per_s"] for r in rows) / len(rows)}), flush=True)


if __name__ == "__main__":
    main()
