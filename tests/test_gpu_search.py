"""GPU: dvc_mcts_search (C++ host tree over the CUDA rollout batches) and the
Python multi-rank driver equal the oracle's flat MCTS exactly (visit and win
table, best move) at reduced budgets (SURVEY §8(c.8) C3 visit-table parity)."""

import json
import os

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

CASES = ["fixtures/c1_d2.json", "fixtures/c2_d2.json", "fixtures/c3_d1.json", "fixtures/xstop_d2.json",
         "fixtures/x3_d1.json", "fixtures/c4_d2.json", "tests/golden/T2c1.json", "tests/golden/E1.json"]


@pytest.fixture(scope="module")
def dvc():
    from paper_2403_10720_b200 import build
    build.build()
    from paper_2403_10720_b200 import dvc as m
    return m


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(p) for p in CASES])
def test_flat_search_equals_oracle(dvc, oracle_lib, path):
    from oracle.search import flat_search
    d = json.load(open(os.path.join(ROOT, path)))
    P = d["rules"]["players"]
    exp_n, n = (24, 64) if P == 4 else (64, 256)
    best_o, stats_o = flat_search(d, exp_n, n, 21)
    st = dvc.encode(d)
    best_g, stats_g = dvc.mcts_search(st, exp_n, n, 21)
    assert [tuple(map(int, t)) for t in stats_g] == stats_o
    assert best_g == best_o
    from paper_2403_10720_b200 import dist
    best_d, stats_d = dist.mcts_search(st, exp_n, n, 21)
    assert stats_d == stats_o and best_d == best_o


DEVICE_CASES = [("fixtures/c3_d1.json", 96, 1000), ("fixtures/c2_d2.json", 80, 4097),
                ("tests/golden/T2c1.json", 300, 128), ("fixtures/x3_d1.json", 70, 333),
                ("fixtures/xsmall_d3.json", 40, 20000), ("fixtures/c4_d2.json", 140, 200)]


@pytest.mark.parametrize("path,exp_n,n", DEVICE_CASES, ids=[os.path.basename(c[0]) for c in DEVICE_CASES])
def test_device_search_loop_equals_host_loop_and_oracle(dvc, oracle_lib, path, exp_n, n):
    """The cooperative flat_search_kernel (search_device=1: UCB1 selection,
    playouts and backpropagation on the GPU, grid barrier per iteration) gives
    the same table as the host loop (search_device=0) and the oracle's
    flat_search, over budgets that run many iterations after the root
    expansion, with n not a multiple of the block and grids of several blocks."""
    from oracle.search import flat_search
    d = json.load(open(os.path.join(ROOT, path)))
    st = dvc.encode(d)
    assert exp_n > len(st.legal_actions())          # iterations remain after the root expansion
    with dvc.options(search_device=1):
        best_dev, stats_dev = dvc.mcts_search(st, exp_n, n, 77)
    with dvc.options(search_device=0):
        best_host, stats_host = dvc.mcts_search(st, exp_n, n, 77)
    stats_dev = [tuple(map(int, t)) for t in stats_dev]
    assert stats_dev == [tuple(map(int, t)) for t in stats_host] and best_dev == best_host
    best_o, stats_o = flat_search(d, exp_n, n, 77)
    assert stats_dev == stats_o and best_dev == best_o
    assert sum(v for _, v, _ in stats_dev) == exp_n * n


def test_search_errors(dvc):
    d = json.load(open(os.path.join(ROOT, "fixtures", "c2_d1.json")))
    st = dvc.encode(d)
    with pytest.raises(dvc.DvcError):
        dvc.mcts_search(st, 0, 10, 1)
    with pytest.raises(dvc.DvcError):
        dvc.mcts_search(st, 4, 10, 1, flat=0, max_depth=9)


PATH_CASES = ["tests/golden/T2c1.json", "fixtures/c2_d2.json", "fixtures/c3_d2.json", "fixtures/x3_d1.json",
              "fixtures/xstop_d1.json", "fixtures/x4mid_d2.json", "fixtures/xsmall_d3.json", "fixtures/xlate_d2.json",
              "fixtures/c4_d5.json"]


@pytest.mark.parametrize("kernel", [0, 1], ids=["refill", "naive"])
@pytest.mark.parametrize("path", PATH_CASES, ids=[os.path.basename(p) for p in PATH_CASES])
def test_path_batches_equal_oracle(dvc, oracle_lib, path, kernel):
    """dvc_rollout_path_ex (forced viewer actions, void playouts) == oracle."""
    import numpy as np
    d = json.load(open(os.path.join(ROOT, path)))
    st = dvc.encode(d)
    L = st.legal_actions()
    STOP = 0xFFFFFFFF
    cons = d["rules"].get("consecutive", 1)
    guesses = [c for c in L if c != STOP]
    paths = [[guesses[0]], [guesses[-1], guesses[0]], [guesses[len(guesses) // 2]] + guesses[:2]]
    codes = guesses[:6] + ([STOP] if cons else [])
    n = 300 if d["rules"]["players"] < 4 else 120
    with dvc.options(kernel=kernel):
        for pth in paths:
            h, v = dvc.rollout_path_ex(st, pth, codes, 13, 5, 7, 7 + n)
            eh, ev = oracle_lib.rollout_path(d, pth, codes, 13, 5, 7, 7 + n)
            assert h.astype(np.int64).tolist() == eh and v.astype(np.int64).tolist() == ev, pth


@pytest.mark.parametrize("path", CASES[:6], ids=[os.path.basename(p) for p in CASES[:6]])
@pytest.mark.parametrize("sdev", [0, 1], ids=["host_tree", "device_tree"])
def test_deep_search_equals_oracle(dvc, oracle_lib, path, sdev):
    from oracle.search import deep_search
    d = json.load(open(os.path.join(ROOT, path)))
    P = d["rules"]["players"]
    exp_n, n = (5, 48) if P == 4 else (8, 128)
    best_o, stats_o = deep_search(d, exp_n, n, 33, max_depth=3)
    st = dvc.encode(d)
    with dvc.options(search_device=sdev):
        best_g, stats_g = dvc.mcts_search(st, exp_n, n, 33, max_depth=3, flat=0)
    assert [tuple(map(int, t)) for t in stats_g] == stats_o
    assert best_g == best_o


DEEP_DEV = [("fixtures/c3_d1.json", 40, 300, 4), ("fixtures/c2_d2.json", 60, 200, 3),
            ("tests/golden/T2c1.json", 50, 100, 4), ("fixtures/xstop_d1.json", 30, 150, 2),
            ("fixtures/x3_d1.json", 20, 100, 4), ("fixtures/c4_d5.json", 12, 60, 3),
            ("fixtures/xsmall_d3.json", 80, 64, 8), ("fixtures/c1_d1.json", 25, 333, 1)]


@pytest.mark.parametrize("path,exp_n,n,depth", DEEP_DEV, ids=[os.path.basename(c[0]) for c in DEEP_DEV])
def test_device_tree_equals_host_tree_and_oracle(dvc, oracle_lib, path, exp_n, n, depth):
    """The cooperative deep_search_kernel (search_device=1: tree in device
    memory, UCB1 descent / expansion / backprop by one warp, batches over the
    grid) reproduces the host tree (search_device=0) and the oracle's
    deep_search exactly, over many iterations, depths 1..8 and void-heavy
    trees."""
    from oracle.search import deep_search
    d = json.load(open(os.path.join(ROOT, path)))
    st = dvc.encode(d)
    with dvc.options(search_device=1):
        best_d, stats_d = dvc.mcts_search(st, exp_n, n, 61, max_depth=depth, flat=0)
    with dvc.options(search_device=0):
        best_h, stats_h = dvc.mcts_search(st, exp_n, n, 61, max_depth=depth, flat=0)
    stats_d = [tuple(map(int, t)) for t in stats_d]
    assert stats_d == [tuple(map(int, t)) for t in stats_h] and best_d == best_h
    best_o, stats_o = deep_search(d, exp_n, n, 61, max_depth=depth)
    assert stats_d == stats_o and best_d == best_o


@pytest.mark.parametrize("flat,seed,sdev", [(1, 1, 0), (1, 2, 1), (0, 3, 0), (0, 4, 1)])
def test_selfplay_equals_oracle(dvc, oracle_lib, flat, seed, sdev):
    """C3 shape (2 players, 26 tiles with jokers): a full self-play game with
    the GPU searches reproduces the oracle's game move for move."""
    from paper_2403_10720_b200.selfplay import play_game
    from oracle.selfplay import play_game as oracle_game
    kw = dict(expansions=6, sims_per_child=64, flat=flat, max_depth=2)
    with dvc.options(search_device=sdev):
        g = play_game(seed, **kw)
    o = oracle_game(seed, **kw)
    assert g == o
    assert g["decisions"] >= 2


def test_concurrent_selfplay_equals_sequential(dvc):
    """Games played on 6 host threads (one CUDA stream each) equal the same
    games played one at a time."""
    from paper_2403_10720_b200.selfplay import play_game, play_games
    kw = dict(expansions=8, sims_per_child=128, flat=1)
    seeds = [11, 12, 13, 14, 15, 16]
    seq = [play_game(s, **kw) for s in seeds]
    assert play_games(seeds, threads=6, **kw) == seq
    kw = dict(expansions=6, sims_per_child=64, flat=0, max_depth=3)
    seq = [play_game(s, **kw) for s in seeds[:3]]
    assert play_games(seeds[:3], threads=3, **kw) == seq


@pytest.mark.parametrize("sdev", [0, 1], ids=["host_loop", "device_loop"])
@pytest.mark.parametrize("path", ["fixtures/c3_d2.json", "fixtures/c2_d1.json", "fixtures/x4mid_d1.json"])
def test_flat_search_flags_equal_oracle(dvc, oracle_lib, path, sdev):
    """Flat search with the informed policy and CRN batches (DESIGN.md §R10,
    §R3) == the oracle's flat_search with the same flags, host and device loops."""
    from oracle.search import flat_search
    d = json.load(open(os.path.join(ROOT, path)))
    st = dvc.encode(d)
    A = len(st.legal_actions())
    exp_n, n = A + 30, 200
    for crn, informed in ((False, True), (True, True), (True, False)):
        best_o, stats_o = flat_search(d, exp_n, n, 5, crn=crn, informed=informed)
        with dvc.options(search_device=sdev):
            best_g, stats_g = dvc.mcts_search(st, exp_n, n, 5, crn=crn, informed=informed)
        assert [tuple(map(int, t)) for t in stats_g] == stats_o and best_g == best_o, (crn, informed)
