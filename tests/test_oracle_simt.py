"""Pins for the SIMT model (oracle/simt.py): the worked examples of SPEC:393-410
and its invariants (monotone masks, efficiency 1 for equal lengths,
efficiency = mean / mean-of-max)."""

import json
import os
import random

from oracle.simt import simulate_warp, simd_efficiency, playout_iterations

from conftest import ROOT


def test_spec_examples():
    assert simulate_warp([4, 4, 4, 4], 4) == [4, 4, 4, 4]
    assert simulate_warp([1, 4], 2) == [2, 1, 1, 1]
    assert simulate_warp([3], 1) == [1, 1, 1]
    assert simd_efficiency([4, 4, 4, 4], 4) == 1.0
    assert simd_efficiency([2, 1, 1, 1], 2) == 0.625


def test_invariants():
    rng = random.Random(4)
    for _ in range(200):
        w = rng.choice([1, 2, 4, 8, 32])
        steps = [rng.randint(1, 30) for _ in range(w)]
        m = simulate_warp(steps, w)
        assert all(a >= b for a, b in zip(m, m[1:]))
        e = simd_efficiency(m, w)
        assert abs(e - (sum(steps) / w) / max(steps)) < 1e-12
    assert simd_efficiency(simulate_warp([7] * 32, 32), 32) == 1.0


def test_playout_lengths_bounded(oracle_lib):
    d = json.load(open(os.path.join(ROOT, "fixtures", "c2_d1.json")))
    codes = oracle_lib.legal(d)
    lens = playout_iterations(d, codes[0], 1, 0, 0, 200)
    # <= 2(|T|-1) decisions (SURVEY §8(c.3) bound) + the start iteration
    assert all(1 <= x <= 2 * 23 + 1 for x in lens)
