"""Pins for deep-tree (path-forced) playouts: exact outcome
distributions by enumeration (oracle/exact.py exact_path, incl. the VOID
probability) on hand-checkable T2 paths; Monte Carlo convergence of the C++
oracle to them; the Python and C++ oracles agree playout for playout."""

import json
import math
import os
from fractions import Fraction

import pytest

from oracle import game as G
from oracle.exact import exact_path

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")
B1, B2, W0, W1 = G.action_code(1, 0, 2), G.action_code(1, 0, 4), G.action_code(1, 1, 1), G.action_code(1, 1, 3)
STOP = G.STOP


def t2():
    return json.load(open(os.path.join(GOLD, "T2c1.json")))


def test_hand_checked_paths():
    """T2 (opponent holds exactly B1, W1): guessing B1 then W1 wins for sure;
    B2 at the root is wrong for sure, the viewer reveals W2 and -- with B0 still
    hidden -- cannot decide again before the opponent, whose turn may end the
    game; W1 then B1 wins for sure."""
    obs = G.Observation.from_json(t2())
    assert exact_path(obs, [B1], W1) == [1, 0, 0]
    assert exact_path(obs, [W1], B1) == [1, 0, 0]
    assert exact_path(obs, [B1, W1], B2) == [0, 0, 1]     # the game is over after two correct guesses
    p = exact_path(obs, [B1], STOP)
    assert sum(p) == 1 and p[2] == 0


@pytest.mark.parametrize("path,code", [([B1], STOP), ([B1], W0), ([B2], W1), ([B2], B1), ([W0], W1)])
def test_mc_converges_to_exact_path(oracle_lib, path, code):
    d = t2()
    ex = exact_path(G.Observation.from_json(d), path, code)
    n = 20000
    hist, voids = oracle_lib.rollout_path(d, path, [code], 3, 17, 0, n)
    got = hist[0] + [voids[0]]
    for p, c in zip(ex, got):
        p = float(p)
        if p in (0.0, 1.0):
            assert c / n == p
        else:
            assert abs(c / n - p) <= 5 * math.sqrt(p * (1 - p) / n)


@pytest.mark.parametrize("name", ["c2_d2", "x3_d1", "xstop_d1", "c3_d2", "x4mid_d2", "xsmall_d3", "xlate_d2"])
def test_python_equals_cpp_path(oracle_lib, name):
    d = json.load(open(os.path.join(ROOT, "fixtures", name + ".json")))
    obs = G.Observation.from_json(d)
    sp = G.DetSpace(obs)
    L = oracle_lib.legal(d)
    path = [L[0], L[-1] if L[-1] != STOP else L[0]]
    codes = L[:4] + ([STOP] if d["rules"]["consecutive"] else [])
    hist, voids = oracle_lib.rollout_path(d, path, codes, 7, 11, 0, 40)
    P = d["rules"]["players"]
    for a, c in enumerate(codes):
        h = [0] * P
        v = 0
        for s in range(40):
            r = G.playout_path(sp, path, c, 7, 11, s)
            if r == G.VOID:
                v += 1
            else:
                h[r] += 1
        assert hist[a] == h and voids[a] == v
