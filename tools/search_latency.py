"""Per-iteration latency of dvc_mcts_search (flat): device-resident UCB loop
(search_device=1) vs host loop (0), over sims per iteration.

    python tools/search_latency.py [fixture]
Prints one JSON line per (search_device, n): ms per decision and the
marginal ms per iteration after the root expansion."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2403_10720_b200 import dvc
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "fixtures", "c3_d1.json")
    d = json.load(open(path))
    st = dvc.encode(d)
    A = len(st.legal_actions())
    for sd in (1, 0):
        with dvc.options(search_device=sd):
            for n in (32, 128, 1024, 4096, 16384):
                res = {}
                for extra in (0, 100):
                    exp_n = A + extra
                    dvc.mcts_search(st, exp_n, n, 1)
                    torch.cuda.synchronize()
                    reps = 10
                    t0 = time.perf_counter()
                    for i in range(reps):
                        dvc.mcts_search(st, exp_n, n, 2 + i)
                    res[extra] = (time.perf_counter() - t0) / reps * 1e3
                print(json.dumps({"search_device": sd, "n": n, "A": A, "ms_root_expansion_only": round(res[0], 4),
                                  "ms_per_iteration": round((res[100] - res[0]) / 100, 5)}), flush=True)


if __name__ == "__main__":
    main()
