"""ms per depth-capped decision (dvc_mcts_search flat=0): host tree vs the
device-resident tree, on a C3 root.   python tools/search_latency_deep.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2403_10720_b200 import dvc
    d = json.load(open(os.path.join(ROOT, "fixtures", "c3_d1.json")))
    st = dvc.encode(d)
    for sd in (0, 1):
        with dvc.options(search_device=sd):
            for exp_n, n in ((64, 1024), (64, 128), (256, 1024)):
                dvc.mcts_search(st, exp_n, n, 1, flat=0, max_depth=4)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for i in range(5):
                    dvc.mcts_search(st, exp_n, n, 2 + i, flat=0, max_depth=4)
                ms = (time.perf_counter() - t0) / 5 * 1e3
                print(json.dumps({"search_device": sd, "expansions": exp_n, "sims_per_child": n,
                                  "ms_per_decision": round(ms, 3), "us_per_iteration": round(1e3 * ms / exp_n, 1)}),
                      flush=True)


if __name__ == "__main__":
    main()
