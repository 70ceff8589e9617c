"""Split the per-call overhead: raw ctypes call of dvc_rollout_batch_async with
prepared arguments vs the Python wrapper."""
import ctypes
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
    L = dvc.lib()
    c = (ctypes.c_uint32 * 1)(codes[0])
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    hp = ctypes.c_void_p(hist.data_ptr())
    res = {}

    def raw(n):
        return L.dvc_rollout_batch_async(ctypes.byref(st._s), c, 1, 1, 0, 0, n, hp, None, 0, sp)

    for name, fn in [("raw_1", lambda: raw(1)), ("raw_1024", lambda: raw(1024)),
                     ("wrapped_1024", lambda: dvc.rollout_batch_async(st, codes[:1], 1, 0, 0, 1024, hist)),
                     ("info", lambda: st.info), ("cur_stream", lambda: torch.cuda.current_stream())]:
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(500):
            fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        res[name] = {"host_us": round(1e6 * (t1 - t0) / 500, 2), "incl_drain_us": round(1e6 * (t2 - t0) / 500, 2)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
