import json, time, glob, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2403_10720_b200 import dvc
fx = sorted(glob.glob("/root/repo/fixtures/*.json"))
ds = [json.load(open(f)) for f in fx]
sts = [dvc.encode(d) for d in ds]
# warm
dvc.rollout_batch_ex(sts[0], sts[0].legal_actions()[:1], 1, 0, 0, 32)
t_new, t_old = [], []
for st in sts[:40]:
    c = st.legal_actions()[:1]
    t0 = time.perf_counter(); dvc.rollout_batch_ex(st, c, 1, 0, 0, 32); t1 = time.perf_counter()
    dvc.rollout_batch_ex(st, c, 2, 0, 0, 32); t2 = time.perf_counter()
    t_new.append(t1 - t0); t_old.append(t2 - t1)
t_new.sort(); t_old.sort()
print("new-state call median us", round(1e6 * t_new[len(t_new)//2], 1), "cached", round(1e6 * t_old[len(t_old)//2], 1))
print("new-state max", round(1e6*t_new[-1],1))
