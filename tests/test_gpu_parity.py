"""GPU parity: the CUDA path (through the C-ABI) against the oracle, bit-exact.

Integer outputs => the bar is equality (SURVEY §8(c.8) "GPU <-> oracle:
bit-identical hist").  Covers every committed fixture (C1-C4 shapes plus the
edge sets) x seeds x both kernels, the hand-worked golden fixtures, schedule
invariance (grid, block, kernel, table vs inline unranking, sim-range splits,
action order/subsets), edge cases (root-terminal playouts, n = 1, the last
sim index 2^32-1, STOP roots, empty pool, consecutive = 0), and the bench's
full-size configuration sampled playout-by-playout against the oracle.
"""

import glob
import json
import os
import random

import numpy as np
import pytest

from conftest import ROOT
from oracle_pool import oracle_hist

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def dvc():
    from paper_2403_10720_b200 import build
    build.build()
    from paper_2403_10720_b200 import dvc as m
    return m


def load(path):
    return json.load(open(path))


FIXTURES = sorted(glob.glob(os.path.join(ROOT, "fixtures", "*.json")))
GOLDEN = sorted(p for p in glob.glob(os.path.join(ROOT, "tests", "golden", "*.json")))


def gpu_hist(dvc, d, codes, seed, node, s0, s1):
    st = dvc.encode(d)
    return dvc.rollout_batch_ex(st, codes, seed, node, s0, s1).astype(np.int64).tolist()


def sims_for(d, codes):
    """Sims per action so the oracle finishes in seconds on the box's cores."""
    P = d["rules"]["players"]
    budget = 60000 if P == 4 else 120000
    return max(50, min(2000, budget // max(1, len(codes))))


_EXP = {}


def expected(d, path, codes, seed, n):
    key = (path, seed, n)
    if key not in _EXP:
        _EXP[key] = oracle_hist(d, codes, seed, 0, 0, n)
    return _EXP[key]


@pytest.mark.parametrize("kernel", [0, 1], ids=["refill", "naive"])
@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p) for p in FIXTURES])
def test_fixture_parity(dvc, oracle_lib, path, kernel):
    d = load(path)
    codes = oracle_lib.legal(d)
    n = sims_for(d, codes)
    for seed in (1, 2, 3):
        exp = expected(d, path, codes, seed, n)
        with dvc.options(kernel=kernel):
            got = gpu_hist(dvc, d, codes, seed, 0, 0, n)
        assert got == exp, (os.path.basename(path), seed)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_golden_parity(dvc, oracle_lib, path):
    d = load(path)
    codes = oracle_lib.legal(d)
    exp = oracle_hist(d, codes, 7, 5, 100, 4100)
    for kernel in (0, 1):
        with dvc.options(kernel=kernel):
            assert gpu_hist(dvc, d, codes, 7, 5, 100, 4100) == exp


def test_golden_forced_results(dvc):
    """E1: every playout wins at the root; E3: B0 always wins, B2 always loses."""
    d = load(os.path.join(ROOT, "tests", "golden", "E1.json"))
    st = dvc.encode(d)
    assert dvc.rollout_batch(st, st.legal_actions(), 100000, 3).tolist() == [100000]
    d = load(os.path.join(ROOT, "tests", "golden", "E3.json"))
    st = dvc.encode(d)
    assert dvc.rollout_batch(st, st.legal_actions(), 100000, 3).tolist() == [100000, 0]


def test_schedule_invariance(dvc):
    d = load(os.path.join(ROOT, "fixtures", "c2_d2.json"))
    st = dvc.encode(d)
    codes = st.legal_actions()
    ref = dvc.rollout_batch_ex(st, codes, 11, 0, 0, 30000)
    configs = [dict(kernel=1), dict(kernel=0, block=32), dict(kernel=0, block=64), dict(kernel=0, block=256),
               dict(kernel=0, grid=1), dict(kernel=0, grid=7), dict(kernel=1, block=1024),
               dict(kernel=1, grid=3, block=64), dict(kernel=1, grid=5, block=7), dict(kernel=1, grid=2, block=1),
               dict(table_cap=0), dict(table_cap=0, kernel=1),
               dict(chunk=100000), dict(chunk=77777, kernel=1)]
    for cfg in configs:
        with dvc.options(**cfg):
            assert (dvc.rollout_batch_ex(st, codes, 11, 0, 0, 30000) == ref).all(), cfg
    for bad in (512, 48):                         # beyond the launch bound / not whole warps
        with dvc.options(kernel=0, block=bad):
            with pytest.raises(dvc.DvcError):
                dvc.rollout_batch_ex(st, codes, 11, 0, 0, 100)
    ref20 = dvc.rollout_batch_ex(st, codes, 11, 0, 0, 20)[:3]
    with dvc.options(chunk=1, grid=2):            # one sim per launch
        assert (dvc.rollout_batch_ex(st, codes[:3], 11, 0, 0, 20) == ref20).all()
    # split sim ranges
    parts = [0, 1, 777, 15000, 30000]
    tot = sum(dvc.rollout_batch_ex(st, codes, 11, 0, a, b) for a, b in zip(parts, parts[1:]))
    assert (tot == ref).all()
    # permuted / subset action lists: keyed by code, so rows follow their codes
    perm = list(range(len(codes)))
    random.Random(3).shuffle(perm)
    got = dvc.rollout_batch_ex(st, [codes[i] for i in perm], 11, 0, 0, 30000)
    assert (got == ref[perm]).all()
    sub = perm[:5]
    assert (dvc.rollout_batch_ex(st, [codes[i] for i in sub], 11, 0, 0, 30000) == ref[sub]).all()


def test_table_vs_inline_unrank_c4(dvc, oracle_lib):
    d = load(os.path.join(ROOT, "fixtures", "c4_d3.json"))
    st = dvc.encode(d)
    codes = st.legal_actions()[::7]
    ref = dvc.rollout_batch_ex(st, codes, 5, 0, 0, 5000)
    with dvc.options(table_cap=0):
        assert (dvc.rollout_batch_ex(st, codes, 5, 0, 0, 5000) == ref).all()
    assert ref.astype(np.int64).tolist() == oracle_hist(d, codes, 5, 0, 0, 5000)


def test_edge_sim_ranges(dvc, oracle_lib):
    d = load(os.path.join(ROOT, "fixtures", "xstop_d1.json"))
    codes = oracle_lib.legal(d)
    assert codes[-1] == 0xFFFFFFFF          # STOP is legal at this root
    for s0, s1 in [(0, 1), (12345, 12346), ((1 << 32) - 300, 1 << 32)]:
        assert gpu_hist(dvc, d, codes, 9, 1, s0, s1) == oracle_hist(d, codes, 9, 1, s0, s1)
    st = dvc.encode(d)
    with pytest.raises(dvc.DvcError):
        dvc.rollout_batch_ex(st, codes, 9, 1, 0, (1 << 32) + 1)
    with pytest.raises(dvc.DvcError):
        dvc.rollout_batch_ex(st, codes, 9, 1, 5, 5)


def test_async_accumulates_and_visits(dvc):
    d = load(os.path.join(ROOT, "fixtures", "c1_d1.json"))
    st = dvc.encode(d)
    codes = st.legal_actions()
    P = st.players
    hist = torch.zeros((len(codes), P), dtype=torch.int64, device="cuda")
    visits = torch.zeros(len(codes), dtype=torch.int64, device="cuda")
    dvc.rollout_batch_async(st, codes, 4, 0, 0, 500, hist, visits)
    dvc.rollout_batch_async(st, codes, 4, 0, 500, 1000, hist, visits)
    torch.cuda.synchronize()
    ref = dvc.rollout_batch_ex(st, codes, 4, 0, 0, 1000)
    assert (hist.cpu().numpy().astype(np.uint64) == ref).all()
    assert visits.cpu().tolist() == [1000] * len(codes)
    assert int(hist.sum()) == 1000 * len(codes)


def _sampled_full_size(dvc, oracle_lib, name, n, samples):
    d = load(os.path.join(ROOT, "fixtures", name))
    st = dvc.encode(d)
    codes = st.legal_actions()
    A, P = len(codes), st.players
    hist = torch.zeros((A, P), dtype=torch.int64, device="cuda")
    win = torch.full((A * n,), 255, dtype=torch.uint8, device="cuda")
    dvc.rollout_trace_async(st, codes, 1, 0, 0, n, hist, win)
    torch.cuda.synchronize()
    w = win.cpu().numpy().reshape(A, n)
    assert (w < P).all()
    h = hist.cpu().numpy()
    for p in range(P):
        assert (h[:, p] == (w == p).sum(axis=1)).all()
    rng = random.Random(17)
    for _ in range(samples):
        a, s = rng.randrange(A), rng.randrange(n)
        wo, _ = oracle_lib.playout(d, codes[a], 1, 0, s)
        assert w[a, s] == wo, (a, s)
    # the untraced launch (the bench's) gives the same counts
    hist2 = torch.zeros_like(hist)
    dvc.rollout_batch_async(st, codes, 1, 0, 0, n, hist2)
    torch.cuda.synchronize()
    assert torch.equal(hist, hist2)
    return d, codes, h


def test_full_size_c2_bench_config(dvc, oracle_lib):
    """BASELINE configs[1]: C2 mid-game, 10^6 playouts per action, 1 B200."""
    d, codes, h = _sampled_full_size(dvc, oracle_lib, "c2_d1.json", 1000000, 3000)
    assert (h.sum(axis=1) == 1000000).all()
    # a contiguous prefix of every action against the all-core oracle
    st = dvc.encode(d)
    assert dvc.rollout_batch_ex(st, codes, 1, 0, 0, 20000).astype(np.int64).tolist() == \
        oracle_hist(d, codes, 1, 0, 0, 20000)


def test_full_size_c4_sampled(dvc, oracle_lib):
    """BASELINE configs[3] shape on one GPU: 4p/26 tiles, ~1e8 playouts per move."""
    _sampled_full_size(dvc, oracle_lib, "c4_d1.json", 1000000, 400)


# ---- common random numbers across actions (DESIGN.md §R3 CRN)
CRN_CASES = ["tests/golden/E2.json", "tests/golden/T1.json", "tests/golden/J1.json", "fixtures/c1_d1.json",
             "fixtures/c2_d3.json", "fixtures/c3_d2.json", "fixtures/x3_d2.json", "fixtures/c4_d3.json",
             "fixtures/xc0_d1.json"]


@pytest.mark.parametrize("kernel", [0, 1], ids=["refill", "naive"])
@pytest.mark.parametrize("path", CRN_CASES, ids=[os.path.basename(p) for p in CRN_CASES])
def test_crn_equals_oracle(dvc, oracle_lib, path, kernel):
    d = load(os.path.join(ROOT, path))
    st = dvc.encode(d)
    codes = st.legal_actions()[:12]
    n = 400 if d["rules"]["players"] < 4 else 150
    exp = oracle_lib.rollout(d, codes, 31, 2, 17, 17 + n, crn=True)
    with dvc.options(kernel=kernel):
        got = dvc.rollout_batch_ex(st, codes, 31, 2, 17, 17 + n, crn=True).astype(np.int64).tolist()
        hist = torch.zeros((len(codes), st.players), dtype=torch.int64, device="cuda")
        dvc.rollout_batch_async(st, codes, 31, 2, 17, 17 + n, hist, crn=True)
        torch.cuda.synchronize()
    assert got == exp
    assert hist.cpu().tolist() == exp
    # a different determinization stream than the default keying
    assert dvc.rollout_batch_ex(st, codes, 31, 2, 17, 17 + n).astype(np.int64).tolist() != exp or len(codes) == 1


def test_crn_e2_complementary_at_full_size(dvc):
    """E2 at 10^6 sims per action: under CRN exactly one of the two guesses
    wins each sim (closed form, tests/test_oracle_crn.py), at any size."""
    d = load(os.path.join(ROOT, "tests", "golden", "E2.json"))
    st = dvc.encode(d)
    codes = st.legal_actions()
    assert len(codes) == 2
    h = dvc.rollout_batch_ex(st, codes, 5, 0, 0, 1000000, crn=True).astype(np.int64)
    assert int(h[0, 0] + h[1, 0]) == 1000000
    assert abs(int(h[0, 0]) - 500000) < 5 * 500                       # p = 1/2, 5 sigma


# ---- informed (order-aware) playout policy
INF_CASES = ["tests/golden/I1.json", "tests/golden/T1.json", "tests/golden/J1.json", "tests/golden/T2c1.json",
             "fixtures/c1_d3.json", "fixtures/c2_d1.json", "fixtures/c3_d1.json", "fixtures/c3_d4.json",
             "fixtures/x3_d1.json", "fixtures/x4mid_d2.json", "fixtures/c4_d1.json", "fixtures/xlate_d1.json",
             "fixtures/xstop_d1.json", "fixtures/xc0_d2.json", "fixtures/x3nj_d1.json", "fixtures/x4jc0_d1.json"]


@pytest.mark.parametrize("kernel", [0, 1], ids=["refill", "naive"])
@pytest.mark.parametrize("path", INF_CASES, ids=[os.path.basename(p) for p in INF_CASES])
def test_informed_equals_oracle(dvc, oracle_lib, path, kernel):
    d = load(os.path.join(ROOT, path))
    st = dvc.encode(d)
    codes = st.legal_actions()
    codes = codes[:6] + codes[-3:] if len(codes) > 9 else codes
    n = 500 if d["rules"]["players"] < 4 else 150
    for crn in (False, True):
        exp = oracle_lib.rollout(d, codes, 8, 1, 3, 3 + n, crn=crn, informed=True)
        with dvc.options(kernel=kernel):
            got = dvc.rollout_batch_ex(st, codes, 8, 1, 3, 3 + n, crn=crn, informed=True).astype(np.int64).tolist()
            hist = torch.zeros((len(codes), st.players), dtype=torch.int64, device="cuda")
            dvc.rollout_batch_async(st, codes, 8, 1, 3, 3 + n, hist, crn=crn, informed=True)
            torch.cuda.synchronize()
        assert got == exp, (path, crn)
        assert hist.cpu().tolist() == exp


def test_informed_i1_exact_at_full_size(dvc):
    """I1 (hand-derived, tests/golden/I1.json): under the informed policy the
    two wrong root guesses lose every playout and the right one wins every
    playout -- at 10^6 sims per action; the plain policy gives 1/4."""
    d = load(os.path.join(ROOT, "tests", "golden", "I1.json"))
    st = dvc.encode(d)
    codes = st.legal_actions()
    n = 1000000
    h = dvc.rollout_batch_ex(st, codes, 4, 0, 0, n, informed=True).astype(np.int64)
    assert h[:, 0].tolist() == [n, 0, 0]
    hp = dvc.rollout_batch_ex(st, codes, 4, 0, 0, n).astype(np.int64)
    for w in hp[1:, 0]:
        assert abs(w / n - 0.25) <= 5 * (0.25 * 0.75 / n) ** 0.5


def test_flags_errors(dvc):
    d = load(os.path.join(ROOT, "fixtures", "c2_d1.json"))
    st = dvc.encode(d)
    codes = st.legal_actions()[:2]
    import ctypes
    L = dvc.lib()
    a = (ctypes.c_uint32 * 2)(*codes)
    h = (ctypes.c_uint64 * (2 * st.players))()
    assert L.dvc_rollout_batch_flags_ex(ctypes.byref(st._s), a, 2, 1, 0, 0, 10, 4, h, -1) == -1   # unknown flag
    with pytest.raises(dvc.DvcError):
        dvc.mcts_search(st, 4, 10, 1, flat=0, informed=True)                   # no path batches with flags
