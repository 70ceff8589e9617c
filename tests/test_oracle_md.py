"""Pins for the fixed-determinization playout of the "md" ablation (DESIGN.md
§R11; "nodes are enriched with information regarding the chosen set
of numbers"): a child (rho, a) plays determinization rho of Det(O), never a
sampled one.

* E2 closed form: the game is decided by the root guess, so under a fixed rho
  the viewer wins all n playouts iff the guessed key is the one unrank(rho)
  puts in the slot, and none otherwise.
* Exact conditionals: on the golden tiny positions, for every rho, the Monte
  Carlo estimate converges to p(a | sigma_rho) computed by full chance
  enumeration (oracle/exact.py) within 5 sigma (equality at 0 and 1), and
  averaging those exact conditionals over rho recovers the golden unconditional
  p(a) the paper-level tests pin.
* Python oracle == C++ oracle, bit-exact, on every golden position.
"""

import math
from fractions import Fraction

import pytest

from oracle import game as G
from oracle.exact import exact_action_fixed
from test_oracle_rules import EXACT, expected_codes, gold


def test_e2_fixed_rho_closed_form(oracle_lib):
    d = gold("E2")
    obs = G.Observation.from_json(d)
    space = G.DetSpace(obs)
    codes = expected_codes(d)
    n = 500
    for rho in range(space.N):
        slot_key = space.unrank(rho)[0]          # the single hidden slot's key under sigma_rho
        hist = oracle_lib.rollout_fixed(d, codes, [rho] * len(codes), 7, 0, 0, n)
        for c, h in zip(codes, hist):
            win = (c & 0xFFFF) == slot_key
            assert h[d["viewer"]] == (n if win else 0)
            assert sum(h) == n


@pytest.mark.parametrize("name", EXACT)
def test_fixed_rho_converges_to_exact_conditional(oracle_lib, name):
    d = gold(name)
    obs = G.Observation.from_json(d)
    space = G.DetSpace(obs)
    codes = expected_codes(d)
    n = 4000
    memo = {}
    v = d["viewer"]
    for rho in range(space.N):
        hist = oracle_lib.rollout_fixed(d, codes, [rho] * len(codes), 99, 3, 0, n)
        for c, h in zip(codes, hist):
            p = float(exact_action_fixed(obs, c, rho, memo)[v])
            est = h[v] / n
            assert sum(h) == n
            if p in (0.0, 1.0):
                assert est == p, (name, rho, c)
            else:
                assert abs(est - p) <= 5 * math.sqrt(p * (1 - p) / n), (name, rho, c, est, p)


@pytest.mark.parametrize("name", EXACT)
def test_exact_conditionals_average_to_golden(name):
    d = gold(name)
    obs = G.Observation.from_json(d)
    space = G.DetSpace(obs)
    memo = {}
    for c, p in zip(expected_codes(d), d["expected"]["p_viewer"]):
        avg = sum(exact_action_fixed(obs, c, r, memo)[obs.viewer] for r in range(space.N)) / space.N
        assert avg == Fraction(p)


@pytest.mark.parametrize("name", EXACT)
def test_fixed_rho_python_equals_cpp(oracle_lib, name):
    d = gold(name)
    obs = G.Observation.from_json(d)
    space = G.DetSpace(obs)
    codes = expected_codes(d)
    rhos = [(i * 7 + 3) % space.N for i in range(len(codes))]
    assert G.rollout_fixed(obs, codes, rhos, 5, 11, 100, 400) == oracle_lib.rollout_fixed(d, codes, rhos, 5, 11, 100, 400)


def test_fixed_rho_rejects_out_of_range(oracle_lib):
    d = gold("E2")
    codes = expected_codes(d)
    with pytest.raises(RuntimeError):
        oracle_lib.rollout_fixed(d, codes[:1], [2], 1, 0, 0, 10)
