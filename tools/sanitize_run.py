"""Small launches of every kernel of libdvc.so, for compute-sanitizer
(VERDICT r01 item 6):

    compute-sanitizer --tool racecheck|synccheck|memcheck|initcheck \
        python tools/sanitize_run.py [--quick]

Covers: rollout_refill_kernel (plain, path, informed, trace modes; small grids
so every warp claims many work batches and drains its ring), the naive
kernel, det_table_kernel, the cooperative flat_search_kernel and
deep_search_kernel (hand-written grid barrier), add_u64_kernel (visits)."""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_2403_10720_b200 import dvc
    n = 300 if args.quick else 1500
    load = lambda p: json.load(open(os.path.join(ROOT, p)))
    for path in ("fixtures/c2_d1.json", "fixtures/c4_d2.json", "fixtures/c3_d1.json", "fixtures/x3_d1.json"):
        d = load(path)
        st = dvc.encode(d)
        codes = st.legal_actions()
        P = st.players
        for kernel, grid in ((0, 2), (0, 0), (1, 3)):
            with dvc.options(kernel=kernel, grid=grid):
                h = torch.zeros((len(codes), P), dtype=torch.int64, device="cuda")
                v = torch.zeros((len(codes),), dtype=torch.int64, device="cuda")
                dvc.rollout_batch_async(st, codes, 3, 0, 0, n, h, v)
                dvc.rollout_batch_async(st, codes, 3, 1, 0, n, h, informed=True)
                w = torch.zeros((len(codes) * n,), dtype=torch.uint8, device="cuda")
                dvc.rollout_trace_async(st, codes, 3, 0, 0, n, h, w)
                dvc.rollout_path_ex(st, [codes[0]], codes[:4], 3, 2, 0, n)
                torch.cuda.synchronize()
                assert int(v.sum()) == len(codes) * n
        with dvc.options(table_cap=0):                     # inline unranking
            dvc.rollout_batch_ex(st, codes, 5, 0, 0, n)
        for sdev in (0, 1):
            with dvc.options(search_device=sdev):
                dvc.mcts_search(st, len(codes) + 6, 64, 7)
                dvc.mcts_search(st, 6, 32, 7, max_depth=3, flat=0)
        print("ok", path, flush=True)
    dvc.shutdown()
    print("sanitize run done")


if __name__ == "__main__":
    main()
