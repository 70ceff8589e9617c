"""Pins for the informed (order-aware) playout policy (SURVEY
§8(f) N4): in a playout every decision is uniform over the guesses whose value
is consistent with the visible order of the target line -- a numbered value
must lie strictly between the nearest revealed numbered tiles left and right of
the slot; a joker value is always kept -- instead of LEGAL.

  * I1 (tests/golden/I1.json): hand-derived lists and exact probabilities
    (plain 1, 1/4, 1/4; informed 1, 0, 0), checked against the exact
    enumerator and the Monte Carlo oracles (Python, C++);
  * on random reachable states (fuzz): the informed list equals a second,
    differently written definition (inserting v at the slot keeps the line's
    revealed numbered keys strictly increasing), is a subset of LEGAL in LEGAL
    order, and contains every hidden slot's true tile;
  * with no revealed tile anywhere the two policies coincide at that state.
"""

import json
import os
import random

import pytest

from conftest import ROOT
from oracle import exact
from oracle import game as G
from oracle import philox as px


def gold(name):
    return json.load(open(os.path.join(ROOT, "tests", "golden", name + ".json")))


def codes_of(d, key):
    R = d["rules"]["ranks"]
    out = []
    for j, pos, col, v in d["expected"][key]:
        c = 0 if col == "B" else 1
        out.append(G.action_code(j, pos, 2 * R + c if v == "J" else 2 * v + c))
    return out


def test_i1_lists():
    d = gold("I1")
    obs = G.Observation.from_json(d)
    assert G.root_legal(obs) == codes_of(d, "legal")
    assert G.root_legal(obs, informed=True) == codes_of(d, "legal_informed")
    assert G.DetSpace(obs).N == d["expected"]["N"]


def test_i1_exact_probabilities():
    from fractions import Fraction
    d = gold("I1")
    obs = G.Observation.from_json(d)
    codes = codes_of(d, "legal")
    assert [exact.exact_action(obs, c)[0] for c in codes] == [Fraction(x) for x in d["expected"]["p_viewer"]]
    assert [exact.exact_action(obs, c, informed=True)[0] for c in codes] == \
        [Fraction(x) for x in d["expected"]["p_viewer_informed"]]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_i1_monte_carlo(oracle_lib, seed):
    """p in {0, 1} => the counts are exact; the plain policy converges to 1/4."""
    d = gold("I1")
    obs = G.Observation.from_json(d)
    codes = codes_of(d, "legal")
    n = 3000
    hi = oracle_lib.rollout(d, codes, seed, 0, 0, n, informed=True)
    assert [h[0] for h in hi] == [n, 0, 0]
    assert G.rollout(obs, codes, seed, 0, 0, 300, informed=True) == oracle_lib.rollout(d, codes, seed, 0, 0, 300,
                                                                                       informed=True)
    hp = oracle_lib.rollout(d, codes, seed, 0, 0, n)
    assert hp[0][0] == n
    for h in hp[1:]:
        assert abs(h[0] / n - 0.25) <= 5 * (0.25 * 0.75 / n) ** 0.5


def _second_definition(game, code):
    """v fits slot pos of line j iff the revealed numbered keys of the line,
    with v put at pos, strictly increase (jokers carry no order)."""
    j, pos, v = G.decode_action(code)
    if game.rules.is_joker(v):
        return True
    seq = []
    for p, (k, r) in enumerate(game.lines[j]):
        if p == pos:
            seq.append(v)
        elif r and not game.rules.is_joker(k):
            seq.append(k)
    return all(a < b for a, b in zip(seq, seq[1:]))


FUZZ = ["c1_d1", "c2_d2", "c3_d1", "c3_d3", "x3_d1", "c4_d1", "x4mid_d1", "xlate_d1", "xstop_d2"]


@pytest.mark.parametrize("name", FUZZ)
def test_informed_list_fuzz(name):
    d = json.load(open(os.path.join(ROOT, "fixtures", name + ".json")))
    obs = G.Observation.from_json(d)
    space = G.DetSpace(obs)
    rng = random.Random(name)
    states = 0
    for _ in range(25):
        game = space.game(space.unrank(rng.randrange(space.N)))
        step = "DECIDE"
        while step != "FINISH":
            if step == "END_TURN":
                game.start_turn(rng.getrandbits(32), rng.getrandbits(32))
            L = game.legal()
            Li = game.legal(informed=True)
            assert Li == [c for c in L if _second_definition(game, c)]
            for c in L:                             # the true tile of every hidden slot stays guessable
                j, pos, v = G.decode_action(c)
                if game.lines[j][pos][0] == v:
                    assert c in Li
            if not any(r for ln in game.lines for _, r in ln):
                assert Li == L
            states += 1
            n = game.n_choices(Li)
            i = px.choose(n, rng.getrandbits(32))
            step = game.apply(G.STOP if i == len(Li) else Li[i])
    assert states > 100


def test_informed_python_equals_cpp(oracle_lib):
    for name in ("c1_d2", "c3_d2", "x3_d2", "c4_d2", "xc0_d1"):
        d = json.load(open(os.path.join(ROOT, "fixtures", name + ".json")))
        obs = G.Observation.from_json(d)
        codes = G.root_legal(obs)[:4]
        n = 40 if d["rules"]["players"] < 4 else 15
        for crn in (False, True):
            assert oracle_lib.rollout(d, codes, 3, 1, 10, 10 + n, crn=crn, informed=True) == \
                G.rollout(obs, codes, 3, 1, 10, 10 + n, crn=crn, informed=True), name
