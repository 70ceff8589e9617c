"""ORACLE (test infrastructure only) -- the flat (root-only) MCTS of
dvc_mcts_search, written plainly in Python on top of the C++ oracle's rollout
(DESIGN.md §R8).  PAPER:112-117 (four MCTS steps), PAPER:180 ("the game
iteratively expands a child node from the root, with subsequent gameplay
unfolding randomly after the initial move"), UCB1 and best-move rules from
SPEC:240-264.
"""

import math

from . import rollout as oracle_rollout, legal as oracle_legal, rollout_fixed as oracle_rollout_fixed, \
    count as oracle_count
from . import philox as px


LN2 = 0.6931471805599453        # the double nearest ln 2


ATANH_C = [1.0 / (2 * k + 1) for k in range(14)]   # 1/(2k+1), each correctly rounded


def ln_series(N):
    """ln N for an integer N >= 1 by a fixed IEEE-double recipe (DESIGN.md §R8,
    reading #28) that the C++ host tree and the CUDA search kernels evaluate
    operation for operation, so all three choose the same UCB1 child:
    N = m 2^e with m in [sqrt(1/2), sqrt(2)), ln N = 2 atanh(z) + e ln2 with
    z = (m - 1)/(m + 1) (|z| < 0.172) and atanh(z) = z * p(z^2), p the
    14-term series sum_k z^(2k) / (2k+1) in Horner form (a multiply, then an
    add, per term; no fused ops).  Accurate to ~1.5 ulp
    (tests/test_oracle_search.py)."""
    m, e = math.frexp(float(N))
    if m < 0.7071067811865476:
        m *= 2.0
        e -= 1
    z = (m - 1.0) / (m + 1.0)
    z2 = z * z
    p = ATANH_C[13]
    for k in range(12, -1, -1):
        p = p * z2 + ATANH_C[k]
    return 2.0 * (z * p) + e * LN2


def ucb1(wins, visits, parent_visits, c):
    """wins/visits + c*sqrt(ln(parent)/visits); unvisited -> +inf.
    ln is ln_series (reading #28), evaluated in this order, no fused ops."""
    if visits == 0:
        return math.inf
    return wins / visits + c * math.sqrt(ln_series(parent_visits) / visits)


def best_child(stats):
    """Most visits, then most wins, then smallest code.
    stats: list of (code, visits, wins)."""
    return min(stats, key=lambda t: (-t[1], -t[2], t[0]))[0]


def flat_search(obs_json, expansions, sims_per_child, seed, c=math.sqrt(2.0), crn=False, informed=False):
    """Returns (best_code, [(code, visits, wins)] in LEGAL order); crn /
    informed select the batch variants (§R10) for every batch."""
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
        h = oracle_rollout(obs_json, [codes[best]], seed, 0, visits[best], visits[best] + sims_per_child,
                           crn=crn, informed=informed)[0]
        # BACKPROPAGATION
        visits[best] += sims_per_child
        wins[best] += h[viewer]
        N += sims_per_child
    stats = list(zip(codes, visits, wins))
    return best_child(stats), stats


def deep_search(obs_json, expansions, sims_per_child, seed, max_depth=4, c=math.sqrt(2.0)):
    """Depth-capped tree over the viewer's guesses,
    written plainly: nodes are dicts; each iteration descends by UCB1, expands
    the leaf with all candidate children in one batch (or re-simulates a leaf at
    max_depth), counts non-void playouts and backpropagates them to the root.
    Returns (best_code, [(code, visits, wins)] of the root's children in LEGAL order)."""
    from . import rollout_path as oracle_rollout_path
    root_codes = oracle_legal(obs_json)
    deep_codes = [x for x in root_codes if x != 0xFFFFFFFF]
    if obs_json["rules"].get("consecutive", 1):
        deep_codes.append(0xFFFFFFFF)
    viewer = obs_json["viewer"]
    nodes = [{"code": None, "depth": 0, "parent": None, "children": [], "expanded": False,
              "visits": 0, "wins": 0, "tried": 0}]
    for _ in range(expansions):
        # SELECTION
        x = 0
        while nodes[x]["expanded"]:
            best = None
            for ch in nodes[x]["children"]:
                node = nodes[ch]
                if node["tried"] > 0 and node["visits"] == 0:
                    continue
                v = math.inf if node["tried"] == 0 else ucb1(node["wins"], node["visits"], nodes[x]["visits"], c)
                if best is None or v > bv or (v == bv and node["code"] < nodes[best]["code"]):
                    best, bv = ch, v
            if best is None:
                break
            x = best
        path = []
        y = x
        while y != 0:
            path.append(nodes[y]["code"])
            y = nodes[y]["parent"]
        path.reverse()
        X = nodes[x]
        if not X["expanded"] and X["depth"] < max_depth and (x == 0 or X["visits"] > 0):
            # EXPANSION of every candidate child, evaluated in one batch
            cand = root_codes if x == 0 else deep_codes
            evaluated = []
            for code in cand:
                nodes.append({"code": code, "depth": X["depth"] + 1, "parent": x, "children": [],
                              "expanded": False, "visits": 0, "wins": 0, "tried": 0})
                X["children"].append(len(nodes) - 1)
                evaluated.append(len(nodes) - 1)
            X["expanded"] = True
            prefix, batch, node_word = path, list(cand), x
        else:
            if x == 0:
                break
            prefix, batch, node_word, evaluated = path[:-1], [X["code"]], X["parent"], [x]
        s0 = nodes[evaluated[0]]["tried"]
        # SIMULATION
        hist, voids = oracle_rollout_path(obs_json, prefix, batch, seed, node_word, s0, s0 + sims_per_child)
        # BACKPROPAGATION
        dv = dw = 0
        for i, e in enumerate(evaluated):
            nodes[e]["tried"] += sims_per_child
            nodes[e]["visits"] += sims_per_child - voids[i]
            nodes[e]["wins"] += hist[i][viewer]
            dv += sims_per_child - voids[i]
            dw += hist[i][viewer]
        y = nodes[evaluated[0]]["parent"]
        while y is not None:
            nodes[y]["visits"] += dv
            nodes[y]["wins"] += dw
            y = nodes[y]["parent"]
    by_code = {nodes[ch]["code"]: (nodes[ch]["visits"], nodes[ch]["wins"]) for ch in nodes[0]["children"]}
    stats = [(code, by_code.get(code, (0, 0))[0], by_code.get(code, (0, 0))[1]) for code in root_codes]
    return best_child(stats), stats


def md_candidates(obs_json, n_det, seed):
    """The md ablation's candidate determinizations: all of
    Det(O) when N <= n_det, else the first n_det distinct rho of the CRN
    determinization blocks of sims 0, 1, ... (node 0), at most 64 n_det draws."""
    N = oracle_count(obs_json)
    if N <= n_det:
        return list(range(N))
    out = []
    for s in range(64 * n_det):
        D = px.det_block(seed, 0, px.CRN_WORD, s)
        r = px.rank64(N, D[0], D[1])
        if r not in out:
            out.append(r)
            if len(out) == n_det:
                break
    return out


def md_search(obs_json, n_det, expansions, sims_per_child, seed, c=math.sqrt(2.0)):
    """The md ablation (PAPER:143 vanilla tree, discarded at
    PAPER:145): flat UCT over children j = i*A + a = (rho_i, LEGAL[a]); child j's
    playouts play determinization rho_i with Philox node 1 + i.  Returns
    (best_code, [(code, visits, wins)] summed over rho_i in LEGAL order, K)."""
    codes = oracle_legal(obs_json)
    viewer = obs_json["viewer"]
    rhos = md_candidates(obs_json, n_det, seed)
    K, A = len(rhos), len(codes)
    visits = [0] * (K * A)
    wins = [0] * (K * A)
    N = 0
    for _ in range(expansions):
        best = None
        for j in range(K * A):
            v = ucb1(wins[j], visits[j], N, c)
            if best is None or v > bv:          # ties -> smallest index
                best, bv = j, v
        i, a = divmod(best, A)
        h = oracle_rollout_fixed(obs_json, [codes[a]], [rhos[i]], seed, 1 + i, visits[best],
                                 visits[best] + sims_per_child)[0]
        visits[best] += sims_per_child
        wins[best] += h[viewer]
        N += sims_per_child
    va = [sum(visits[i * A + a] for i in range(K)) for a in range(A)]
    wa = [sum(wins[i * A + a] for i in range(K)) for a in range(A)]
    stats = list(zip(codes, va, wa))
    return best_child(stats), stats, K
