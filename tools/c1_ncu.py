"""One C1 decision batch (c1_d1, all legal x 1000) on the default (auto) path,
for ncu: python tools/c1_ncu.py"""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_10720_b200 import dvc
d = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures", "c1_d1.json")))
st = dvc.encode(d); codes = st.legal_actions()
hist = torch.zeros((len(codes), 2), dtype=torch.int64, device="cuda")
for i in range(3):
    dvc.rollout_batch_async(st, codes, 1 + i, 0, 0, 1000, hist)
torch.cuda.synchronize()
