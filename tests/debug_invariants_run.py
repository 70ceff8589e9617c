"""Runs under DVC_DEBUG=1 (libdvc_debug.so): every committed fixture through
both kernels (plain, deep-tree path and informed/CRN batches), then prints the device-side
invariant counters as JSON.  Driven by tests/test_gpu_debug.py."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    assert os.environ.get("DVC_DEBUG") == "1"
    from paper_2403_10720_b200 import dvc
    assert dvc.LIB_PATH.endswith("libdvc_debug.so")
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    for path in sorted(glob.glob(os.path.join(ROOT, "fixtures", "*.json"))):
        d = json.load(open(path))
        st = dvc.encode(d)
        codes = st.legal_actions()
        for kernel in (0, 1):
            with dvc.options(kernel=kernel):
                dvc.rollout_batch_ex(st, codes, 31, 0, 0, n)
                guesses = [c for c in codes if c != 0xFFFFFFFF]
                dvc.rollout_path_ex(st, [guesses[0]], codes[:8], 31, 1, 0, n // 10)
                dvc.rollout_batch_ex(st, codes, 32, 0, 0, n // 4, crn=True, informed=True)
        # the trace mode (per-playout winner writes) and a 2-block grid, where
        # every warp claims many work batches (bounds codes 11-13)
        import torch
        m = max(1, n // 10)
        hist = torch.zeros((len(codes), st.players), dtype=torch.int64, device="cuda")
        win = torch.zeros((len(codes) * m,), dtype=torch.uint8, device="cuda")
        with dvc.options(kernel=0, grid=2):
            dvc.rollout_trace_async(st, codes, 33, 0, 7, 7 + m, hist, win)
            dvc.rollout_batch_ex(st, codes, 34, 0, 0, m)
        torch.cuda.synchronize()
    print(json.dumps({"counters": list(dvc.debug_counters())}))


if __name__ == "__main__":
    main()
