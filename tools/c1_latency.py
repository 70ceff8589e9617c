"""C1 latency breakdown (one decision: encode, legal actions, blocking rollout
with a cached plan, async launch + sync, device span).  python tools/c1_latency.py [fixture]"""
import json, time, sys, glob
sys.path.insert(0, "/root/repo")
import torch
from paper_2403_10720_b200 import dvc
d = json.load(open("/root/repo/fixtures/" + (sys.argv[1] if len(sys.argv) > 1 else "c1_d1.json")))
st = dvc.encode(d); codes = st.legal_actions()
for _ in range(20): dvc.rollout_batch(st, codes, 1000, 99)
def med(f, n=200):
    ts = []
    for i in range(n):
        t0 = time.perf_counter(); f(i); ts.append(time.perf_counter() - t0)
    ts.sort(); return round(1e6 * ts[len(ts)//2], 1)
print("encode us", med(lambda i: dvc.encode(d)))
print("legal us", med(lambda i: st.legal_actions()))
print("rollout_batch (cached plan) us", med(lambda i: dvc.rollout_batch(st, codes, 1000, 1 + i)))
hist = torch.zeros((len(codes), 2), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
def k(i):
    dvc.rollout_batch_async(st, codes, 1 + i, 0, 0, 1000, hist); torch.cuda.synchronize()
print("async+sync us", med(k))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts=[]
for i in range(100):
    e0.record(s); dvc.rollout_batch_async(st, codes, 1 + i, 0, 0, 1000, hist); e1.record(s); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)*1000)
ts.sort(); print("device span us", round(ts[50],1), "A", len(codes))
for opt in ("plan_cache",):
    v = dvc.get_option(opt) if hasattr(dvc, "get_option") else None
    print(opt, v)
for kern in (0, 1):
    for blk in (32, 64, 128):
        with dvc.options(kernel=kern, block=blk):
            for _ in range(5): k(0)
            ts = []
            for i in range(100):
                e0.record(s); dvc.rollout_batch_async(st, codes, 1 + i, 0, 0, 1000, hist); e1.record(s); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)*1000)
            ts.sort(); print("kernel", kern, "block", blk, "device span us", round(ts[50], 1), "blocking us", med(lambda i: dvc.rollout_batch(st, codes, 1000, 1 + i), 100))
