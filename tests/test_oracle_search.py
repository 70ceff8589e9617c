"""Pins for the oracle's flat MCTS (oracle/search.py): the
worked UCB1 and best-move examples of SPEC:246-248 and SPEC:262-264, budget
conservation, the forced endgame E1, and convergence to the exact best action
(oracle/exact.py) on T2."""

import json
import math
import os
from fractions import Fraction

from oracle.search import ucb1, best_child, flat_search

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")


def test_ucb1_spec_examples():
    assert abs(ucb1(5, 10, 100, math.sqrt(2)) - (0.5 + math.sqrt(2 * math.log(100) / 10))) < 1e-15
    assert abs(ucb1(5, 10, 100, math.sqrt(2)) - 1.4597) < 1e-4
    assert ucb1(0, 0, 10, 0.7) == math.inf
    assert ucb1(10, 10, 10, 1.3) == 1.0 + 1.3 * math.sqrt(math.log(10) / 10)


def test_best_child_spec_examples():
    assert best_child([(1, 700, 0), (2, 300, 300)]) == 1
    assert best_child([(1, 500, 300), (2, 500, 200)]) == 1
    assert best_child([(9, 500, 300), (2, 500, 300)]) == 2                # smallest code on a full tie
    assert best_child([(1, 7000, 0), (2, 3000, 3000)]) == 1               # SPEC:264 (scaling)


def test_forced_endgame(oracle_lib):
    d = json.load(open(os.path.join(GOLD, "E1.json")))
    best, stats = flat_search(d, 5, 100, 3)
    assert len(stats) == 1 and best == stats[0][0]
    assert stats[0][1] == 500 and stats[0][2] == 500                       # win rate 1.0


def test_budget_conservation_and_exact_best(oracle_lib):
    d = json.load(open(os.path.join(GOLD, "T2c1.json")))
    best, stats = flat_search(d, 40, 200, 9)
    assert sum(v for _, v, _ in stats) == 40 * 200
    exact = [Fraction(x) for x in d["expected"]["p_viewer"]]
    best_p = max(exact)
    codes = [c for c, _, _ in stats]
    assert exact[codes.index(best)] == best_p


def test_deep_depth1_equals_flat(oracle_lib):
    """max_depth 1: the root expansion batch + re-simulation of UCB-selected
    root children is exactly flat UCB1 with A - 1 more iterations."""
    from oracle.search import deep_search
    for name in ("fixtures/c2_d2.json", "fixtures/xstop_d1.json", "tests/golden/T2c1.json"):
        d = json.load(open(os.path.join(ROOT, name)))
        A = len(oracle_lib.legal(d))
        assert deep_search(d, 9, 50, 4, max_depth=1) == flat_search(d, A + 8, 50, 4)


def test_deep_search_finds_exact_best(oracle_lib):
    from oracle.search import deep_search
    d = json.load(open(os.path.join(GOLD, "T2c1.json")))
    best, stats = deep_search(d, 12, 200, 9, max_depth=3)
    exact = [Fraction(x) for x in d["expected"]["p_viewer"]]
    assert exact[[c for c, _, _ in stats].index(best)] == max(exact)
    d = json.load(open(os.path.join(GOLD, "E1.json")))
    best, stats = deep_search(d, 4, 100, 3)
    assert stats[0][1] == stats[0][2] > 0                    # forced win, no voids at depth 1


def test_ln_series_accuracy_and_special_values():
    """ln_series (DESIGN.md §R8 reading #28) against a 50-digit decimal ln:
    within 2 ulp everywhere sampled; exact 0 at N = 1; k*ln2 at N = 2^k;
    increasing on 1..10^5."""
    import math
    import random
    from decimal import Decimal, getcontext
    from oracle.search import ln_series, LN2
    getcontext().prec = 50
    assert ln_series(1) == 0.0
    for k in range(1, 63):
        assert ln_series(1 << k) == k * LN2
    rng = random.Random(3)
    for N in list(range(2, 2000)) + [rng.randrange(2, 1 << 52) for _ in range(5000)]:
        a = ln_series(N)
        ref = Decimal(N).ln()
        assert abs(Decimal(a) - ref) <= 2 * Decimal(math.ulp(float(ref))), N
    prev = -1.0
    for N in range(1, 100001):
        v = ln_series(N)
        assert v > prev
        prev = v
