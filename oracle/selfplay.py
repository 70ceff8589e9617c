"""ORACLE (test infrastructure only): self-play with the oracle's rules
(oracle/game.py) and the oracle's searches (oracle/search.py), following the
referee protocol of DESIGN.md §S (deal by random.Random(seed).shuffle, draws
by rng.randrange on the sorted pool, joker gaps by rng.randrange(len + 1)), so
a product self-play game (paper_2403_10720_b200/selfplay.py) must reproduce
the same move list."""

import random

from .game import Game, Rules, NONE
from .fixtures import observe
from .search import flat_search, deep_search


def _draw(game, rng):
    game.pend, game.corr = NONE, 0
    if not game.pool:
        return
    t = game.pool.pop(rng.randrange(len(game.pool)))
    if game.rules.is_joker(t):
        game.insert_joker(game.g, t, rng.randrange(len(game.lines[game.g]) + 1))
    else:
        game.insert_numbered(game.g, t)
    game.pend = t


def play_game(seed, players=2, ranks=12, jokers=1, consecutive=1, per=4, expansions=64, sims_per_child=1024,
              max_depth=4, flat=1, max_decisions=500):
    rules = Rules(players, ranks, jokers, consecutive)
    rng = random.Random(seed)
    T = rules.tiles()
    rng.shuffle(T)
    lines = []
    for p in range(players):
        hand = T[p * per:(p + 1) * per]
        jk = sorted(k for k in hand if rules.is_joker(k))
        num = sorted(k for k in hand if not rules.is_joker(k))
        lines.append([[k, False] for k in jk + num])
    game = Game(rules, lines, sorted(T[players * per:]), 0, NONE, 0)
    _draw(game, rng)
    moves = []
    for i in range(max_decisions):
        obs = observe(game, game.g)
        s = seed * 1000003 + i
        if flat:
            code, _ = flat_search(obs, expansions, sims_per_child, s)
        else:
            code, _ = deep_search(obs, expansions, sims_per_child, s, max_depth=max_depth)
        mover = game.g
        j, pos, v = code >> 24, (code >> 16) & 0xFF, code & 0xFFFF
        correct = code != 0xFFFFFFFF and game.lines[j][pos][0] == v
        out = game.apply(code)
        moves.append((mover, code, correct))
        if out == "FINISH":
            return {"winner": game.winner(), "moves": moves, "decisions": len(moves)}
        if out == "END_TURN":
            game.g = game.next_mover()
            _draw(game, rng)
    raise RuntimeError("game did not finish")
