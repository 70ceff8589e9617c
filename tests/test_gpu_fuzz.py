"""GPU parity on seeded random positions: breadth beyond the committed
fixtures.  Rule variants drawn at random (2-4 players, 3-12 ranks, jokers on or
off, consecutive on or off), deals of 1-5 tiles each, 0-6 random turns, STOP
roots; random seeds and node ids (both ends of the stream key and of the
counter's node bits, §R3) and sim ranges up to the last index 2^32 - 1.  Every
legal action, both kernels, plus CRN and informed batches on a subset: the
CUDA path through the C-ABI against the C++ oracle, bit-exact.  The positions
come from the oracle-side generator (oracle/fixtures.py), built in the test."""

import random

import numpy as np
import pytest

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


def random_cases(n, seed):
    from oracle.fixtures import make_position
    from oracle.game import Rules
    rng = random.Random(seed)
    cases = []
    while len(cases) < n:
        P = rng.choice([2, 2, 3, 4])
        R = rng.randint(3, 12)
        J = rng.randint(0, 1)
        C = rng.randint(0, 1)
        T = 2 * R + 2 * J
        per_max = min(5, (T - 1) // P)
        if per_max < 1:
            continue
        per = rng.randint(1, per_max)
        turns = rng.randint(0, 6)
        extra = 1 if (C and rng.random() < 0.3) else 0
        d = make_position(Rules(players=P, ranks=R, jokers=J, consecutive=C), per, rng.randrange(1 << 30), turns,
                          extra, max_attempts=50)
        if d is None:
            continue
        cases.append(d)
    return cases


CASES = random_cases(48, 20261018)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_random_position_parity(dvc, oracle_lib, i):
    d = CASES[i]
    rng = random.Random(1000 + i)
    st = dvc.encode(d)
    codes = st.legal_actions()
    seed = rng.getrandbits(64)
    node = rng.choice([0, 1, rng.getrandbits(14), rng.getrandbits(32)])
    n = 64
    s0 = rng.choice([0, rng.getrandbits(31), (1 << 32) - n])
    exp = oracle_hist(d, codes, seed, node, s0, s0 + n)
    for kernel in (0, 1):
        with dvc.options(kernel=kernel):
            got = dvc.rollout_batch_ex(st, codes, seed, node, s0, s0 + n).astype(np.int64).tolist()
        assert got == exp, "kernel %d, case %d (%s)" % (kernel, i, d["rules"])


def _oracle_flags(d, codes, seed, node, s0, s1, crn, informed):
    import oracle
    return oracle.rollout(d, codes, seed, node, s0, s1, crn=crn, informed=informed)


@pytest.mark.parametrize("i", range(0, len(CASES), 3))
def test_random_position_variants(dvc, oracle_lib, i):
    """CRN and informed batches on every third random position."""
    d = CASES[i]
    rng = random.Random(2000 + i)
    st = dvc.encode(d)
    codes = st.legal_actions()
    seed, node, n = rng.getrandbits(64), rng.getrandbits(32), 48
    for crn, informed in ((True, False), (False, True)):
        exp = _oracle_flags(d, codes, seed, node, 0, n, crn, informed)
        got = dvc.rollout_batch_ex(st, codes, seed, node, 0, n, crn=crn, informed=informed).astype(np.int64).tolist()
        assert got == exp, "crn=%s informed=%s case %d (%s)" % (crn, informed, i, d["rules"])
