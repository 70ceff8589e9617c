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


def test_search_errors(dvc):
    d = json.load(open(os.path.join(ROOT, "fixtures", "c2_d1.json")))
    st = dvc.encode(d)
    with pytest.raises(dvc.DvcError):
        dvc.mcts_search(st, 0, 10, 1)
    with pytest.raises(dvc.DvcError):
        dvc.mcts_search(st, 4, 10, 1, flat=0)
