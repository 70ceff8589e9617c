"""ORACLE (test infrastructure only) -- the flat (root-only) MCTS of
dvc_mcts_search, written plainly in Python on top of the C++ oracle's rollout
(DESIGN.md §R8).  PAPER:112-117 (four MCTS steps), PAPER:180 ("the game
iteratively expands a child node from the root, with subsequent gameplay
unfolding randomly after the initial move"), UCB1 and best-move rules from
SPEC:240-264.
"""

import math

from . import rollout as oracle_rollout, legal as oracle_legal


def ucb1(wins, visits, parent_visits, c):
    """wins/visits + c*sqrt(ln(parent)/visits); unvisited -> +inf."""
    if visits == 0:
        return math.inf
    return wins / visits + c * math.sqrt(math.log(parent_visits) / visits)


def best_child(stats):
    """Most visits, then most wins, then smallest code.
    stats: list of (code, visits, wins)."""
    return min(stats, key=lambda t: (-t[1], -t[2], t[0]))[0]


def flat_search(obs_json, expansions, sims_per_child, seed, c=math.sqrt(2.0)):
    """Returns (best_code, [(code, visits, wins)] in LEGAL order)."""
    codes = oracle_legal(obs_json)
    viewer = obs_json["viewer"]
    visits = [0] * len(codes)
    wins = [0] * len(codes)
    N = 0
    for _ in range(expansions):
        # SELECTION: max UCB1, ties -> smallest code
        best = None
        for a in range(len(codes)):
            v = ucb1(wins[a], visits[a], N, c)
            if best is None or v > bv or (v == bv and codes[a] < codes[best]):
                best, bv = a, v
        # SIMULATION of sims [visits, visits + n) of that child (node 0)
        h = oracle_rollout(obs_json, [codes[best]], seed, 0, visits[best], visits[best] + sims_per_child)[0]
        # BACKPROPAGATION
        visits[best] += sims_per_child
        wins[best] += h[viewer]
        N += sims_per_child
    stats = list(zip(codes, visits, wins))
    return best_child(stats), stats
