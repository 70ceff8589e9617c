"""Pins for the rules and the playout (§R5; §II-A,
PAPER:114):

  * hand-worked fixtures (tests/golden): legal-guess lists and exact win
    probabilities, computed by oracle/exact.py's chance enumeration;
  * SPEC:130 worked example (32 legal guesses);
  * Monte Carlo convergence of the C++ oracle to the exact values;
  * the two oracle implementations (Python list rules, C++ list rules) agree
    playout-for-playout on every committed fixture;
  * invariant fuzz of random games.
"""

import glob
import json
import math
import os
import random
from fractions import Fraction

import pytest

from oracle import game as G
from oracle.exact import exact_action
from oracle.fixtures import _deal, _start_turn

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")
EXACT = ["E1", "E2", "E3", "T1", "T1c0", "T2c0", "T2c1", "J1"]


def gold(name):
    return json.load(open(os.path.join(GOLD, name + ".json")))


def expected_codes(d):
    R = d["rules"]["ranks"]
    out = []
    for j, pos, col, v in d["expected"]["legal"]:
        c = 0 if col == "B" else 1
        key = 2 * R + c if v == "J" else 2 * v + c
        out.append(G.action_code(j, pos, key))
    return out


@pytest.mark.parametrize("name", EXACT)
def test_golden_legal(oracle_lib, name):
    d = gold(name)
    exp = expected_codes(d)
    assert G.root_legal(G.Observation.from_json(d)) == exp
    assert oracle_lib.legal(d) == exp


def test_spec130_legal_count(oracle_lib):
    d = gold("S130")
    assert len(oracle_lib.legal(d)) == 32
    assert len(G.root_legal(G.Observation.from_json(d))) == 32


@pytest.mark.parametrize("name", EXACT)
def test_golden_exact_probabilities(name):
    d = gold(name)
    obs = G.Observation.from_json(d)
    got = [exact_action(obs, c)[obs.viewer] for c in expected_codes(d)]
    assert got == [Fraction(x) for x in d["expected"]["p_viewer"]]


@pytest.mark.parametrize("name", EXACT)
def test_mc_converges_to_exact(oracle_lib, name):
    """|hist/n - p| <= 5 sqrt(p(1-p)/n); equality when p in {0, 1}."""
    d = gold(name)
    codes = expected_codes(d)
    n = 20000
    hist = oracle_lib.rollout(d, codes, 12345, 0, 0, n)
    for a, p in zip(hist, d["expected"]["p_viewer"]):
        p = float(Fraction(p))
        est = a[d["viewer"]] / n
        assert sum(a) == n
        if p in (0.0, 1.0):
            assert est == p
        else:
            assert abs(est - p) <= 5 * math.sqrt(p * (1 - p) / n)


def tiny_cases():
    """Tiny 2- and 3-player positions for exact-vs-MC on random structure."""
    from oracle.fixtures import make_position
    out = []
    for s, (P, R, jok, per, turns) in enumerate([(2, 3, 0, 2, 0), (2, 3, 1, 2, 1), (3, 2, 0, 1, 0),
                                                   (3, 2, 1, 1, 0), (2, 2, 1, 2, 0), (2, 3, 0, 2, 1)]):
        out.append(make_position(G.Rules(P, R, jok, 1), per, 900 + s, turns))
        out.append(make_position(G.Rules(P, R, jok, 0), per, 900 + s, turns))
    return out


@pytest.mark.parametrize("idx", range(12))
def test_mc_converges_to_exact_random_tiny(oracle_lib, idx):
    d = tiny_cases()[idx]
    obs = G.Observation.from_json(d)
    codes = oracle_lib.legal(d)[:6]
    n = 20000
    hist = oracle_lib.rollout(d, codes, 777, 0, 0, n)
    memo = {}
    for c, h in zip(codes, hist):
        ex = exact_action(obs, c, memo)
        assert sum(ex) == 1
        for w in range(obs.rules.P):
            p = float(ex[w])
            est = h[w] / n
            if p in (0.0, 1.0):
                assert est == p
            else:
                assert abs(est - p) <= 5 * math.sqrt(p * (1 - p) / n) + 1e-12


FIXTURES = sorted(glob.glob(os.path.join(ROOT, "fixtures", "*.json")))


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p) for p in FIXTURES])
def test_python_oracle_equals_cpp_oracle(oracle_lib, path):
    d = json.load(open(path))
    obs = G.Observation.from_json(d)
    codes = oracle_lib.legal(d)
    assert codes == G.root_legal(obs)
    codes = codes[:: max(1, len(codes) // 4)]
    n = 6
    assert oracle_lib.rollout(d, codes, 99, 3, 1000, 1000 + n) == G.rollout(obs, codes, 99, 3, 1000, 1000 + n)


def _check_invariants(game, T):
    R = game.rules
    keys = sorted([k for ln in game.lines for k, _ in ln] + game.pool)
    assert keys == T                                          # tile conservation
    for ln in game.lines:
        nums = [k for k, _ in ln if not R.is_joker(k)]
        assert nums == sorted(nums)                           # sortedness


@pytest.mark.parametrize("rk", [(2, 12, 0, 1), (2, 12, 1, 1), (2, 12, 0, 0), (3, 12, 1, 1), (4, 12, 1, 1)])
def test_invariant_fuzz(rk):
    rules = G.Rules(*rk)
    T = rules.tiles()
    per = 3 if rules.P == 4 else 4
    rng = random.Random(hash(rk) & 0xFFFF)
    for game_no in range(150):
        game = _deal(rules, per, rng)
        _start_turn(game, rng, first=True)
        guesses = 0
        revealed = 0
        while True:
            _check_invariants(game, T)
            L = game.legal()
            n = game.n_choices(L)
            assert n >= 1 and len(L) >= 1
            # every action targets a hidden slot of an alive opponent, and the
            # true tile of every hidden slot of every alive opponent is in LEGAL
            for a in L:
                j, pos, v = G.decode_action(a)
                assert j != game.g and game.alive(j) and not game.lines[j][pos][1]
            Ls = set(L)
            for j in range(rules.P):
                if j == game.g or not game.alive(j):
                    continue
                for pos, (k, r) in enumerate(game.lines[j]):
                    if not r:
                        assert G.action_code(j, pos, k) in Ls
            i = rng.randrange(n)
            a = G.STOP if i == len(L) else L[i]
            st = game.apply(a)
            now = sum(1 for ln in game.lines for _, r in ln if r)
            if a != G.STOP:
                guesses += 1
                assert now == revealed + 1                    # exactly one reveal per guess
            else:
                assert now == revealed
            revealed = now
            if st == "FINISH":
                break
            if st == "END_TURN":
                game.start_turn(rng.getrandbits(32), rng.getrandbits(32))
        assert guesses <= len(T) - 1
        w = game.winner()
        for p in range(rules.P):
            hidden = sum(1 for _, r in game.lines[p] if not r)
            assert (hidden >= 1) == (p == w)
