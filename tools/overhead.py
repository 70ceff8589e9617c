"""Per-call overhead of the C-ABI entry points (tiny batches), for the C1/C3
latency analysis.   python tools/overhead.py"""
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
    codes = st.legal_actions()
    hist = torch.zeros((1, st.players), dtype=torch.int64, device="cuda")
    res = {}
    for name, n, fn in [
        ("encode", 2000, lambda: dvc.encode(d)),
        ("ex_1x1", 300, lambda: dvc.rollout_batch_ex(st, codes[:1], 1, 0, 0, 1)),
        ("ex_1x1024", 300, lambda: dvc.rollout_batch_ex(st, codes[:1], 1, 0, 0, 1024)),
        ("async_1x1024+sync", 300, lambda: (dvc.rollout_batch_async(st, codes[:1], 1, 0, 0, 1024, hist),
                                            torch.cuda.synchronize())),
        ("async_1x1024_nosync", 300, lambda: dvc.rollout_batch_async(st, codes[:1], 1, 0, 0, 1024, hist)),
    ]:
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        res[name] = round(1e6 * (time.perf_counter() - t0) / n, 2)
    for kern in (0, 1):
        with dvc.options(kernel=kern):
            ts = []
            for _ in range(50):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dvc.rollout_batch_async(st, codes[:1], 1, 0, 0, 1024, hist)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1000)
            res["device_us_1x1024_kernel%d" % kern] = round(min(ts), 2)
    print(json.dumps({"us_per_call": res}))


if __name__ == "__main__":
    main()
