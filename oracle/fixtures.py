"""ORACLE-side seeded position generator (test infrastructure only).

Writes the committed fixtures/*.json: root observations shaped like the paper's
workloads (SURVEY.md §8(d) "Synthetic inputs"), each with the full
hidden truth next to it (rollouts never read `truth`).  Both the oracle and the
CUDA path read these files, so the generator's own RNG (Python's
random.Random(deal_seed)) plays no part in parity.

Recipe:
  * deal: uniform shuffle of T, `per` tiles each, lines sorted (dealt jokers go
    leftmost);
  * `turns` turns of uniform-random play (draw, then uniform decisions from
    LEGAL + STOP-when-allowed, the PAPER:114 policy), redrawn from the next seed
    offset if the game ends;
  * the next player draws -> root at AwaitGuess, viewer = that player;
  * optionally continue the root turn with `extra_correct` correct guesses
    (consecutive rules) so the root has correct_this_turn >= 1 and STOP is legal.

Usage:  python -m oracle.fixtures [outdir]
"""

import json
import os
import random
import sys

from .game import Rules, Game, NONE, STOP, colour


def _deal(rules, per, rng):
    T = rules.tiles()
    rng.shuffle(T)
    lines = []
    for p in range(rules.P):
        hand = T[p * per:(p + 1) * per]
        jok = sorted(k for k in hand if rules.is_joker(k))
        num = sorted(k for k in hand if not rules.is_joker(k))
        lines.append([[k, False] for k in jok + num])
    pool = sorted(T[rules.P * per:])
    return Game(rules, lines, pool, 0, NONE, 0)


def _start_turn(game, rng, first=False):
    if not first:
        game.start_turn(rng.getrandbits(32), gap_word=rng.getrandbits(32))
    else:  # seat 0's first turn: draw without advancing the mover
        game.pend, game.corr = NONE, 0
        if game.pool:
            from .philox import choose
            t = game.pool.pop(choose(len(game.pool), rng.getrandbits(32)))
            if game.rules.is_joker(t):
                game.insert_joker(game.g, t, choose(len(game.lines[game.g]) + 1, rng.getrandbits(32)))
            else:
                game.insert_numbered(game.g, t)
            game.pend = t


def _play_turn(game, rng):
    """Decisions of one turn after the draw; returns the final step."""
    while True:
        L = game.legal()
        n = game.n_choices(L)
        i = rng.randrange(n)
        a = STOP if i == len(L) else L[i]
        st = game.apply(a)
        if st != "DECIDE":
            return st


def observe(game, viewer):
    R = game.rules
    lines = []
    for p, ln in enumerate(game.lines):
        out = []
        for k, r in ln:
            c = colour(k)
            if R.is_joker(k):
                v = "J"
            else:
                v = k >> 1
            if p != viewer and not r:
                v = None
            out.append({"color": "B" if c == 0 else "W", "value": v, "revealed": bool(r)})
        lines.append(out)
    pending = -1
    if game.pend != NONE:
        for idx, (k, r) in enumerate(game.lines[viewer]):
            if k == game.pend:
                pending = idx
    truth = []
    for ln in game.lines:
        truth.append([{"color": "B" if colour(k) == 0 else "W",
                       "value": "J" if R.is_joker(k) else k >> 1, "revealed": bool(r)} for k, r in ln])
    return {"rules": {"players": R.P, "ranks": R.R, "jokers": R.jokers, "consecutive": R.consecutive},
            "viewer": viewer, "lines": lines, "pool_size": len(game.pool), "pending": pending,
            "correct_this_turn": game.corr, "truth": truth}


def make_position(rules, per, deal_seed, turns, extra_correct=0, until_pool_empty=False, max_attempts=None):
    """max_attempts: give up (return None) after that many redraws (tests'
    random positions; the committed fixtures use the unbounded default)."""
    attempt = 0
    while True:
        if max_attempts is not None and attempt >= max_attempts:
            return None
        rng = random.Random(deal_seed * 1000003 + attempt)
        attempt += 1
        game = _deal(rules, per, rng)
        _start_turn(game, rng, first=True)
        ok = True
        played = 0
        while played < turns or (until_pool_empty and (game.pool or game.pend != NONE)):
            st = _play_turn(game, rng)
            played += 1
            if st == "FINISH":
                ok = False
                break
            _start_turn(game, rng)
        if not ok:
            continue
        # root turn: optionally make correct guesses first (consecutive rules)
        good = True
        for _ in range(extra_correct):
            L = game.legal()
            truthful = [a for a in L if game.lines[a >> 24][(a >> 16) & 0xFF][0] == (a & 0xFFFF)]
            a = truthful[rng.randrange(len(truthful))]
            if game.apply(a) != "DECIDE":
                good = False
                break
        if not good:
            continue
        return observe(game, game.g)


CONFIGS = {
    # name: (rules kwargs, per, turns, extra_correct, until_pool_empty, seeds)
    "c1": (dict(players=2, ranks=12, jokers=0, consecutive=1), 4, 0, 0, False, range(1, 9)),
    "c2": (dict(players=2, ranks=12, jokers=0, consecutive=1), 4, 8, 0, False, range(1, 9)),
    "c3": (dict(players=2, ranks=12, jokers=1, consecutive=1), 4, 0, 0, False, range(1, 5)),
    "c4": (dict(players=4, ranks=12, jokers=1, consecutive=1), 3, 0, 0, False, range(1, 9)),
    # extra parity cases (edge structure): 3 players mid-game with jokers,
    # empty pool (late game), STOP-legal roots, the PAPER:153 variant
    "x3": (dict(players=3, ranks=12, jokers=1, consecutive=1), 4, 6, 0, False, range(1, 5)),
    "xlate": (dict(players=2, ranks=12, jokers=1, consecutive=1), 4, 0, 0, True, range(1, 5)),
    "xstop": (dict(players=2, ranks=12, jokers=1, consecutive=1), 4, 4, 1, False, range(1, 5)),
    "xc0": (dict(players=2, ranks=12, jokers=0, consecutive=0), 4, 8, 0, False, range(1, 5)),
    "x4mid": (dict(players=4, ranks=12, jokers=1, consecutive=1), 3, 10, 0, False, range(1, 5)),
    "xsmall": (dict(players=3, ranks=4, jokers=1, consecutive=1), 2, 2, 0, False, range(1, 5)),
    # every kernel instantiation (players x jokers x consecutive) gets fixtures
    "x3nj": (dict(players=3, ranks=12, jokers=0, consecutive=1), 4, 5, 0, False, range(1, 4)),
    "x4nj": (dict(players=4, ranks=12, jokers=0, consecutive=0), 3, 6, 0, False, range(1, 4)),
    "x3c0": (dict(players=3, ranks=12, jokers=1, consecutive=0), 4, 4, 0, False, range(1, 4)),
    "x2jc0": (dict(players=2, ranks=12, jokers=1, consecutive=0), 4, 6, 0, False, range(1, 4)),
    "x4njc1": (dict(players=4, ranks=12, jokers=0, consecutive=1), 3, 2, 0, False, range(1, 4)),
    "x3njc0": (dict(players=3, ranks=12, jokers=0, consecutive=0), 4, 3, 0, False, range(1, 4)),
    "x4jc0": (dict(players=4, ranks=12, jokers=1, consecutive=0), 3, 3, 0, False, range(1, 4)),
}


def generate(outdir):
    os.makedirs(outdir, exist_ok=True)
    names = []
    for name, (rk, per, turns, extra, until_empty, seeds) in CONFIGS.items():
        for s in seeds:
            pos = make_position(Rules(**rk), per, s, turns, extra, until_empty)
            pos["recipe"] = {"config": name, "deal_seed": s, "tiles_each": per, "turns": turns,
                             "extra_correct": extra, "until_pool_empty": until_empty,
                             "generator": "oracle/fixtures.py (random.Random(deal_seed*1000003+attempt))"}
            fn = "%s_d%d.json" % (name, s)
            with open(os.path.join(outdir, fn), "w") as f:
                json.dump(pos, f, indent=None, separators=(",", ":"))
                f.write("\n")
            names.append(fn)
    return names


if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "fixtures")
    print("\n".join(generate(out)))
