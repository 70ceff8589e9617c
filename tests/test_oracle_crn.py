"""Pins for the common-random-numbers variant (DESIGN.md §R3 "CRN", SURVEY
§8(f) N4): with crn the determinization block of sim s is keyed by CRN_WORD
instead of the action code, so all actions of a batch play against the same
hidden-tile assignment for each s.

E2 (tests/golden/E2.json) decides the game at the root: the
opponent's only tile is B1 or B2, a correct guess wins at once and a wrong one
eliminates the viewer.  Under CRN, for every s exactly one of the two guesses
wins, so wins(B1) + wins(B2) = n exactly, and wins(B2) counts the sims whose
rank rho = rank64(2, D.x, D.y) is 0 (canonical order §R4: delta(slot = B2) =
(0,0,0,1) < delta(slot = B1) = (0,1,0,0) over U = {W0, B1, W1, B2})."""

import json
import os

import pytest

from conftest import ROOT
from oracle import game as G
from oracle import philox as px

STOP = 0xFFFFFFFF


def load(name):
    return json.load(open(os.path.join(ROOT, name)))


def code(target, pos, key):
    return (target << 24) | (pos << 16) | key


@pytest.mark.parametrize("seed", [1, 7, 0xDEADBEEF12345678])
def test_e2_crn_complementary_and_closed_form(oracle_lib, seed):
    d = load("tests/golden/E2.json")
    b1, b2 = code(1, 0, 2), code(1, 0, 4)
    n = 4000
    h = oracle_lib.rollout(d, [b1, b2], seed, 3, 100, 100 + n, crn=True)
    w1, w2 = h[0][0], h[1][0]
    assert w1 + w2 == n                       # exactly one guess is right for each sim
    assert h[0][0] + h[0][1] == n and h[1][0] + h[1][1] == n
    rho0 = sum(1 for s in range(100, 100 + n)
               if px.rank64(2, *px.det_block(seed, 3, px.CRN_WORD, s)[:2]) == 0)
    assert w2 == rho0 and w1 == n - rho0
    # without CRN the two actions draw independent determinizations
    h2 = oracle_lib.rollout(d, [b1, b2], seed, 3, 100, 100 + n)
    assert h2[0][0] + h2[1][0] != n


def test_crn_word_is_not_an_action_code():
    assert px.CRN_WORD != STOP and (px.CRN_WORD >> 24) > 3


@pytest.mark.parametrize("name", ["tests/golden/T1.json", "tests/golden/T2c1.json", "tests/golden/J1.json",
                                  "fixtures/c1_d1.json", "fixtures/x3_d1.json", "fixtures/c4_d1.json"])
def test_crn_python_equals_cpp(oracle_lib, name):
    d = load(name)
    obs = G.Observation.from_json(d)
    codes = G.root_legal(obs)[:5]
    n = 60 if d["rules"]["players"] < 4 else 20
    assert oracle_lib.rollout(d, codes, 5, 2, 40, 40 + n, crn=True) == G.rollout(obs, codes, 5, 2, 40, 40 + n,
                                                                                   crn=True)


def test_crn_rows_independent_of_the_list(oracle_lib):
    d = load("fixtures/c1_d2.json")
    codes = G.root_legal(G.Observation.from_json(d))
    full = oracle_lib.rollout(d, codes, 9, 0, 0, 300, crn=True)
    for i in (0, len(codes) // 2, len(codes) - 1):
        assert oracle_lib.rollout(d, [codes[i]], 9, 0, 0, 300, crn=True)[0] == full[i]
