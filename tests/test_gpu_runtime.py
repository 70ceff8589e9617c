"""GPU runtime behaviour of the C-ABI scratch: plan/table cache eviction,
dvc_shutdown and lazy re-creation, concurrent launches on several CUDA
streams (each launch owns its work counter), table cap boundaries, and the
launch counter the bench reports."""

import glob
import json
import os

import numpy as np
import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def dvc():
    from paper_2403_10720_b200 import build
    build.build()
    from paper_2403_10720_b200 import dvc as m
    return m


FIX = sorted(glob.glob(os.path.join(ROOT, "fixtures", "*.json")))


def test_plan_cache_eviction_and_shutdown(dvc, oracle_lib):
    # more distinct states than the 16-entry plan cache, twice over
    ds = [json.load(open(p)) for p in FIX[:20]]
    for rnd in range(2):
        for d in ds:
            st = dvc.encode(d)
            codes = st.legal_actions()[:3]
            got = dvc.rollout_batch_ex(st, codes, 5, 0, 0, 64).astype(np.int64).tolist()
            assert got == oracle_lib.rollout(d, codes, 5, 0, 0, 64)
        dvc.shutdown()                      # frees every scratch; the next call re-creates it


def test_concurrent_streams(dvc):
    ds = [json.load(open(os.path.join(ROOT, "fixtures", n))) for n in ("c2_d1.json", "c3_d2.json", "x3_d1.json")]
    sts = [dvc.encode(d) for d in ds]
    ref = [dvc.rollout_batch_ex(st, st.legal_actions(), 3, 0, 0, 20000) for st in sts]
    streams = [torch.cuda.Stream() for _ in sts]
    hists = [torch.zeros((len(st.legal_actions()), st.players), dtype=torch.int64, device="cuda") for st in sts]
    for rep in range(3):
        for h in hists:
            h.zero_()
        torch.cuda.synchronize()
        for st, s, h in zip(sts, streams, hists):
            dvc.rollout_batch_async(st, st.legal_actions(), 3, 0, 0, 20000, h, stream=s)
        torch.cuda.synchronize()
        for h, r in zip(hists, ref):
            assert (h.cpu().numpy().astype(np.uint64) == r).all()


def test_eviction_while_launches_in_flight(dvc):
    """More distinct states than the plan cache holds, launched asynchronously
    on four streams without synchronising: evicted plans must stay intact
    until every launch reading them has finished (per-stream use events and
    the zombie list), and their buffers are reused only then.  Every result
    equals the same batch run alone."""
    ds = [json.load(open(p)) for p in FIX[:48]]
    sts = [dvc.encode(d) for d in ds]
    codes = [st.legal_actions()[:4] for st in sts]
    ref = [dvc.rollout_batch_ex(st, c, 9, 0, 0, 3000) for st, c in zip(sts, codes)]
    dvc.shutdown()
    streams = [torch.cuda.Stream() for _ in range(4)]
    hists = [torch.zeros((len(c), st.players), dtype=torch.int64, device="cuda") for st, c in zip(sts, codes)]
    torch.cuda.synchronize()
    for rep in range(2):
        for i, (st, c, h) in enumerate(zip(sts, codes, hists)):
            dvc.rollout_batch_async(st, c, 9, 0, 0, 3000, h, stream=streams[i % 4])
        torch.cuda.synchronize()
        for h, r in zip(hists, ref):
            assert (h.cpu().numpy().astype(np.uint64) == (rep + 1) * r).all()


def test_table_cap_boundary(dvc):
    d = json.load(open(os.path.join(ROOT, "fixtures", "c1_d5.json")))
    st = dvc.encode(d)
    N = st.info["n_det"]
    codes = st.legal_actions()[:4]
    ref = dvc.rollout_batch_ex(st, codes, 8, 0, 0, 3000)
    for cap in (N, N - 1, 1, 0):
        with dvc.options(table_cap=cap):
            assert (dvc.rollout_batch_ex(st, codes, 8, 0, 0, 3000) == ref).all(), cap


def test_launch_count(dvc):
    d = json.load(open(os.path.join(ROOT, "fixtures", "c2_d1.json")))
    st = dvc.encode(d)
    codes = st.legal_actions()
    hist = torch.zeros((len(codes), 2), dtype=torch.int64, device="cuda")
    dvc.rollout_batch_async(st, codes, 1, 0, 0, 100, hist)      # plan cached
    torch.cuda.synchronize()
    dvc.launch_count(reset=True)
    dvc.rollout_batch_async(st, codes, 1, 0, 0, 100, hist)
    torch.cuda.synchronize()
    assert dvc.launch_count() == 1
    with dvc.options(plan_cache=0):
        dvc.launch_count(reset=True)
        dvc.rollout_batch_async(st, codes, 1, 0, 0, 100, hist)
        torch.cuda.synchronize()
        assert dvc.launch_count() == 2                            # + det_table_kernel
