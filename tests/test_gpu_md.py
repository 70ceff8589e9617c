"""GPU parity of the md ablation (PAPER:143 vanilla tree):
fixed-determinization batches (dvc_rollout_batch_fixed_ex) bit-exact against
the oracle on fixtures of every shape and both kernels, and the md search
(dvc_md_search) choosing the same children with the same counts as the
oracle's md search."""

import json
import os
import random

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


def fx(name):
    sub = "tests/golden" if name[0] in "ETJIS" else "fixtures"
    return json.load(open(os.path.join(ROOT, sub, name + ".json")))


@pytest.mark.parametrize("kernel", [0, 1], ids=["refill", "naive"])
@pytest.mark.parametrize("name", ["T2c1", "J1", "c1_d2", "c2_d1", "c3_d1", "c4_d2", "x3_d1", "xc0_d1"])
def test_fixed_batches_equal_oracle(dvc, oracle_lib, name, kernel):
    d = fx(name)
    st = dvc.encode(d)
    codes = st.legal_actions()
    N = oracle_lib.count(d)
    rng = random.Random(hash(name) & 0xFFFF)
    # every action once, plus repeats of the first under other determinizations
    acts = list(codes) + [codes[0]] * 3
    rhos = [rng.randrange(N) for _ in acts]
    seed, node = rng.getrandbits(64), rng.getrandbits(32)
    n = 300 if d["rules"]["players"] < 4 else 100
    exp = oracle_lib.rollout_fixed(d, acts, rhos, seed, node, 0, n)
    with dvc.options(kernel=kernel):
        got = dvc.rollout_batch_fixed_ex(st, acts, rhos, seed, node, 0, n).astype(np.int64).tolist()
    assert got == exp


def test_fixed_rho_errors(dvc, oracle_lib):
    d = fx("c2_d1")
    st = dvc.encode(d)
    codes = st.legal_actions()
    N = oracle_lib.count(d)
    with pytest.raises(dvc.DvcError) as e:
        dvc.rollout_batch_fixed_ex(st, codes[:2], [0, N], 1, 0, 0, 10)
    assert e.value.code == -1
    with pytest.raises(ValueError):
        dvc.rollout_batch_fixed_ex(st, codes[:2], [0], 1, 0, 0, 10)


@pytest.mark.parametrize("name,n_det,extra", [("T2c1", 8, 30), ("c3_d2", 4, 25), ("c2_d3", 3, 20), ("x3_d2", 2, 10)])
def test_md_search_equals_oracle(dvc, oracle_lib, name, n_det, extra):
    from oracle.search import md_search as oracle_md
    d = fx(name)
    st = dvc.encode(d)
    A = len(st.legal_actions())
    N = oracle_lib.count(d)
    K = min(N, n_det)
    expansions = K * A + extra              # the batched expansion, then UCB1 iterations
    best, table, kd = dvc.md_search(st, n_det, expansions, 64, 99)
    obest, otable, ok = oracle_md(d, n_det, expansions, 64, 99)
    assert kd == ok == K
    assert [tuple(t) for t in table] == [tuple(t) for t in otable]
    assert best == obest
    assert sum(t[1] for t in table) == expansions * 64
