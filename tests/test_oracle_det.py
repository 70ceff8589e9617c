"""Pins for the determinization sampler ("A set of
these plausible numbers is randomly selected for each simulation"):

  * the DP count N and unrank(rho) of both oracle implementations equal a
    brute-force enumeration of every injective colour- and order-consistent
    assignment, sorted by the canonical decision vector delta;
  * observe(sigma) == O for every sigma;
  * the hand-worked counts of tests/golden (E1-E3, T1, T2, J1);
  * uniformity: chi-square over the N categories of rank64(N, D.x, D.y).
"""

import itertools
import json
import os
import random

import pytest

from oracle import philox as px
from oracle.fixtures import make_position
from oracle.game import DetSpace, Observation, Rules

from conftest import ROOT


def brute_force(d):
    """Every consistent assignment, as (delta, {hs_index: key}), sorted by delta.
    Written from the definitions of SURVEY.md §8(c.4), independently of
    oracle/game.py's DP."""
    r = d["rules"]
    R, P, jok = r.get("ranks", 12), r["players"], r.get("jokers", 0)
    g0 = d["viewer"]

    def key(t):
        c = 0 if t["color"] == "B" else 1
        return None if t["value"] is None else (2 * R + c if t["value"] == "J" else 2 * t["value"] + c)

    T = list(range(2 * R + (2 if jok else 0)))
    known = {key(t) for t in d["lines"][g0]}
    for p in range(P):
        if p != g0:
            known |= {key(t) for t in d["lines"][p] if t["revealed"]}
    U = [k for k in T if k not in known]
    HS = []  # (offset d, seat j, line index, colour)
    for dd in range(1, P):
        j = (g0 + dd) % P
        for i, t in enumerate(d["lines"][j]):
            if not t["revealed"]:
                HS.append((dd, j, i, 0 if t["color"] == "B" else 1))
    out = []
    for perm in itertools.permutations(U, len(HS)):
        if any((k & 1) != h[3] for k, h in zip(perm, HS)):
            continue
        lines = {j: [key(t) for t in d["lines"][j]] for j in range(P) if j != g0}
        for k, (dd, j, i, c) in zip(perm, HS):
            lines[j][i] = k
        ok = True
        for j, ln in lines.items():
            nums = [k for k in ln if k < 2 * R]
            if any(a >= b for a, b in zip(nums, nums[1:])):
                ok = False
        if not ok:
            continue
        if len(U) - len(HS) != d["pool_size"]:
            continue
        assign = dict(zip(range(len(HS)), perm))
        delta = []
        if jok:
            for J in (2 * R, 2 * R + 1):
                if J not in U:
                    continue
                same = [h for h in range(len(HS)) if HS[h][3] == (J & 1)]
                o = 0
                for n_, h in enumerate(same):
                    if assign[h] == J:
                        o = 1 + n_
                delta.append(o)
        for u in U:
            if u >= 2 * R:
                continue
            dd = 0
            for h, k in assign.items():
                if k == u:
                    dd = HS[h][0]
            delta.append(dd)
        out.append((tuple(delta), assign))
    out.sort(key=lambda x: x[0])
    return out


def small_positions():
    cases = []
    rng = random.Random(11)
    for n in range(36):
        P = rng.choice([2, 2, 3])
        R = rng.choice([3, 4, 5])
        jok = rng.choice([0, 1])
        per = 2 if P == 3 else rng.choice([2, 3])
        if P * per + 1 > 2 * R + 2 * jok:
            per = 2
        turns = rng.choice([0, 1, 2, 3])
        try:
            cases.append(make_position(Rules(P, R, jok, 1), per, 100 + n, turns))
        except Exception:
            continue
    # larger N: openings with more ranks (brute force stays < ~1e5 permutations)
    for n in range(12):
        P = [2, 3, 4][n % 3]
        R = 6 if P < 4 else 5
        jok = (n // 3) % 2
        cases.append(make_position(Rules(P, R, jok, 1), 2, 500 + n, 0))
    return cases


SMALL = small_positions()


@pytest.mark.parametrize("idx", range(len(SMALL)))
def test_count_and_unrank_equal_brute_force(oracle_lib, idx):
    d = SMALL[idx]
    bf = brute_force(d)
    space = DetSpace(Observation.from_json(d))
    assert space.N == len(bf) >= 1
    assert oracle_lib.count(d) == len(bf)
    for rho, (delta, assign) in enumerate(bf):
        assert space.unrank(rho) == assign, (rho, delta)
        cpp = oracle_lib.unrank(d, rho)
        assert cpp == [assign[h] for h in range(len(assign))]


@pytest.mark.parametrize("idx", range(0, len(SMALL), 3))
def test_observe_of_determinization_is_observation(idx):
    """observe(det) == obs, and the truth is one of the elements."""
    d = SMALL[idx]
    obs = Observation.from_json(d)
    space = DetSpace(obs)
    truth_found = False
    R = obs.rules
    truth = [[R.key_of(t["color"], t["value"]) for t in ln] for ln in d["truth"]]
    for rho in range(space.N):
        g = space.game(space.unrank(rho))
        for p, ln in enumerate(g.lines):
            assert len(ln) == len(obs.lines[p])
            for (k, r), (c, ok, orv) in zip(ln, obs.lines[p]):
                assert (k & 1) == c and r == orv
                if ok is not None:
                    assert k == ok
        assert len(g.pool) == d["pool_size"]
        alltiles = sorted([k for ln in g.lines for k, _ in ln] + g.pool)
        assert alltiles == R.tiles()
        if [[k for k, _ in ln] for ln in g.lines] == truth:
            truth_found = True
    assert truth_found


GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.mark.parametrize("name", ["E1", "E2", "E3", "T1", "T2c0", "T2c1", "J1", "S130"])
def test_golden_counts(oracle_lib, name):
    d = json.load(open(os.path.join(GOLD, name + ".json")))
    exp = d["expected"]
    if "N" in exp:
        assert DetSpace(Observation.from_json(d)).N == exp["N"]
        assert oracle_lib.count(d) == exp["N"]
    if name == "S130":
        from math import comb
        assert oracle_lib.count(d) == comb(8, 4)  # 4 of the 8 remaining blacks, sorted


def test_j1_unrank_order(oracle_lib):
    """J1: rho=0 <-> B1 in the slot, rho=1 <-> JB."""
    d = json.load(open(os.path.join(GOLD, "J1.json")))
    assert oracle_lib.unrank(d, 0) == [2]   # B1 = 2*1+0
    assert oracle_lib.unrank(d, 1) == [4]   # JB = 2R = 4


def test_sampler_chi_square():
    """uniform over Det(O); chi-square at alpha = 0.01 over N categories
    of rho = rank64(N, D.x, D.y), D the determinization block."""
    from scipy.stats import chi2
    d = json.load(open(os.path.join(ROOT, "fixtures", "c1_d1.json")))
    N = DetSpace(Observation.from_json(d)).N
    n = 60000
    counts = [0] * N
    for s in range(n):
        D = px.det_block(3, 0, 0x01000002, s)
        counts[px.rank64(N, D[0], D[1])] += 1
    e = n / N
    stat = sum((c - e) ** 2 / e for c in counts)
    assert stat < chi2.ppf(0.99, N - 1)
