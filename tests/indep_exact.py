"""A SECOND, independently written exact evaluator of the estimand p_w(a)
(SURVEY.md §8(c.0)(i)), for pinning the oracle -- test infrastructure only.

It imports nothing from `oracle/` and nothing from the product: it is written
from the prose of SURVEY.md §8(c.1), (c.2), (c.4) and (c.5) (= DESIGN.md §R1,
§R2, §R4, §R5), with a different representation from `oracle/game.py` so that a
slip in either one shows up as a disagreement:

  * a line is NOT a list of tiles: it is (nums, jokers) -- the holder's numbered
    keys as a sorted tuple, and the held jokers as (key, jslot) in line order,
    jslot = #numbered tiles left of the joker.  The tile list
    is materialised from it when a position is needed;
  * inserting a numbered key t follows §8(c.2) literally: i = #numbered keys of
    the holder below t, every joker with jslot > i moves up by one (so t lands
    RIGHT of a joker in its gap);
  * a drawn joker J at gap gamma in [0, len]: no other joker ->
    jslot = gamma; else, with the other joker at line index lam, gamma <= lam
    -> jslot = gamma, J before it; gamma > lam -> jslot = gamma - 1, J after it;
  * revealed tiles are one global frozenset of keys (keys are unique);
  * Det(O) is enumerated by brute force over all colour-preserving injective
    fillings of the hidden opponent slots, filtered by strict increase of the
    numbered keys along each opponent line (§8(c.4) "consistent assignment"),
    each weighted 1/N -- no DP, no canonical order (the estimand does not need
    one);
  * the next mover is the first ALIVE seat of g+1, g+2, ... (mod P) (PAPER:106
    "the turn passes to the next gambler", SPEC:186 round-robin skipping the
    eliminated);
  * the decision list is LEGAL(g) (opponents in seat order after g, alive
    only; hidden positions left to right; values of the slot's colour in
    ascending key order, not in g's hand, not revealed) plus STOP last when
    consecutive and >= 1 correct guess this turn;
  * a correct guess reveals the target and, under consecutive
    rules, the mover decides again (PAPER:106 vs PAPER:153); a wrong guess
    reveals the mover's pending drawn tile if it is still hidden, else the
    mover's leftmost hidden tile; the game ends when at
    most one player has a hidden tile ("last gambler standing").

Exact rationals (fractions.Fraction); only tiny tile sets.
"""

import itertools
import random
from fractions import Fraction
from functools import lru_cache

STOP = 0xFFFFFFFF


def _key(rules, color, value):
    c = 0 if color in ("B", 0) else 1
    if value == "J":
        return 2 * rules["ranks"] + c
    return 2 * int(value) + c


class Rules:
    def __init__(self, d):
        self.P = d["players"]
        self.R = d.get("ranks", 12)
        self.jok = d.get("jokers", 0)
        self.cons = d.get("consecutive", 1)
        self.JB = 2 * self.R
        self.T = tuple(range(2 * self.R + (2 if self.jok else 0)))

    def joker(self, k):
        return k >= self.JB


# ---------------------------------------------------------------- lines as (nums, jokers)

def line_from_keys(rules, keys):
    """(nums, jokers) of a line given as its keys in line order."""
    nums, jokers = [], []
    for k in keys:
        if rules.joker(k):
            jokers.append((k, len(nums)))
        else:
            nums.append(k)
    assert list(nums) == sorted(nums)
    return (tuple(nums), tuple(jokers))


def materialise(line):
    nums, jokers = line
    out = []
    for i in range(len(nums) + 1):
        for k, js in jokers:
            if js == i:
                out.append(k)
        if i < len(nums):
            out.append(nums[i])
    return out


def insert_numbered(line, t):
    nums, jokers = line
    i = sum(1 for x in nums if x < t)
    jokers = tuple((k, js + 1 if js > i else js) for k, js in jokers)
    return (tuple(sorted(nums + (t,))), jokers)


def insert_joker(line, J, gamma):
    nums, jokers = line
    if not jokers:
        return (nums, ((J, gamma),))
    assert len(jokers) == 1
    (Jo, jso), = jokers
    lam = materialise(line).index(Jo)
    if gamma <= lam:
        return (nums, ((J, gamma), (Jo, jso)))
    return (nums, ((Jo, jso), (J, gamma - 1)))


# ---------------------------------------------------------------- game state
# state = (lines: tuple per seat, revealed: frozenset, pool: tuple sorted, g, pend, corr)

def alive(state, p):
    lines, rev = state[0], state[1]
    return any(k not in rev for k in materialise(lines[p]))


def n_alive(state, P):
    return sum(1 for p in range(P) if alive(state, p))


def legal(rules, state):
    lines, rev, _, g, _, _ = state
    own = set(materialise(lines[g]))
    out = []
    for d in range(1, rules.P):
        j = (g + d) % rules.P
        if not alive(state, j):
            continue
        for pos, k in enumerate(materialise(lines[j])):
            if k in rev:
                continue
            for v in rules.T:                     # ascending keys: numbered, then the joker
                if (v & 1) == (k & 1) and v not in own and v not in rev:
                    out.append((j << 24) | (pos << 16) | v)
    return out


def apply(rules, state, code):
    """-> (state, "FINISH" | "DECIDE" | "END_TURN")."""
    lines, rev, pool, g, pend, corr = state
    if code == STOP:
        return state, "END_TURN"
    j, pos, v = code >> 24, (code >> 16) & 0xFF, code & 0xFFFF
    t = materialise(lines[j])[pos]
    if t == v:
        st = (lines, rev | {t}, pool, g, pend, corr + 1)
        if n_alive(st, rules.P) <= 1:
            return st, "FINISH"
        return st, ("DECIDE" if rules.cons else "END_TURN")
    if pend is not None and pend not in rev:
        r = pend
    else:
        r = next(k for k in materialise(lines[g]) if k not in rev)
    st = (lines, rev | {r}, pool, g, pend, corr)
    return st, ("FINISH" if n_alive(st, rules.P) <= 1 else "END_TURN")


def next_mover(rules, state):
    g = state[3]
    for d in range(1, rules.P + 1):
        p = (g + d) % rules.P
        if alive(state, p):
            return p
    raise AssertionError("nobody alive")


def turn_starts(rules, state):
    """[(probability, state)] after END_TURN: next alive mover, uniform draw,
    a drawn joker at a uniform gap."""
    lines, rev, pool, g, pend, corr = state
    g2 = next_mover(rules, state)
    if not pool:
        return [(Fraction(1), (lines, rev, pool, g2, None, 0))]
    out = []
    for t in pool:
        rest = tuple(x for x in pool if x != t)
        if rules.joker(t):
            L = len(materialise(lines[g2]))
            for gamma in range(L + 1):
                nl = lines[:g2] + (insert_joker(lines[g2], t, gamma),) + lines[g2 + 1:]
                out.append((Fraction(1, len(pool) * (L + 1)), (nl, rev, rest, g2, t, 0)))
        else:
            nl = lines[:g2] + (insert_numbered(lines[g2], t),) + lines[g2 + 1:]
            out.append((Fraction(1, len(pool)), (nl, rev, rest, g2, t, 0)))
    return out


def winner(rules, state):
    w = [p for p in range(rules.P) if alive(state, p)]
    assert len(w) == 1
    return w[0]


def make_value(rules):
    @lru_cache(maxsize=None)
    def value(state, step):
        """Exact winner distribution (tuple over seats) after a decision."""
        if step == "FINISH":
            out = [Fraction(0)] * rules.P
            out[winner(rules, state)] = Fraction(1)
            return tuple(out)
        branches = turn_starts(rules, state) if step == "END_TURN" else [(Fraction(1), state)]
        total = [Fraction(0)] * rules.P
        for pr, st in branches:
            L = legal(rules, st)
            choices = L + ([STOP] if rules.cons and st[5] >= 1 else [])
            for a in choices:
                st2, step2 = apply(rules, st, a)
                v = value(st2, step2)
                for w in range(rules.P):
                    total[w] += pr * Fraction(1, len(choices)) * v[w]
        return tuple(total)
    return value


# ---------------------------------------------------------------- observations

def determinizations(d):
    """All full states consistent with the observation (brute force), at the root."""
    rules = Rules(d["rules"])
    g0 = d["viewer"]
    obs = []
    for line in d["lines"]:
        obs.append([(0 if t["color"] == "B" else 1,
                     None if t.get("value") is None else _key(d["rules"], t["color"], t["value"]),
                     bool(t.get("revealed", False))) for t in line])
    known = {k for _, k, _ in obs[g0]} | {k for p in range(rules.P) for _, k, r in obs[p] if r}
    U = [k for k in rules.T if k not in known]
    slots = [(p, i, c) for p in range(rules.P) if p != g0 for i, (c, k, r) in enumerate(obs[p]) if not r]
    out = []
    for fill in itertools.permutations(U, len(slots)):
        if any((k & 1) != c for k, (_, _, c) in zip(fill, slots)):
            continue
        keys = [[k for _, k, _ in line] for line in obs]
        for k, (p, i, _) in zip(fill, slots):
            keys[p][i] = k
        ok = True
        for p in range(rules.P):
            nums = [k for k in keys[p] if not rules.joker(k)]
            if any(a >= b for a, b in zip(nums, nums[1:])):
                ok = False
        pool = tuple(sorted(set(U) - set(fill)))
        if not ok or len(pool) != d["pool_size"]:
            continue
        lines = tuple(line_from_keys(rules, keys[p]) for p in range(rules.P))
        rev = frozenset(k for p in range(rules.P) for (_, _, r), k in zip(obs[p], keys[p]) if r)
        pend = keys[g0][d["pending"]] if d.get("pending", -1) >= 0 else None
        out.append((lines, rev, pool, g0, pend, d.get("correct_this_turn", 0)))
    return rules, out


def root_legal(d):
    """LEGAL(g0) from the observation alone (a hidden opponent tile only
    contributes its colour) plus STOP when allowed."""
    rules = Rules(d["rules"])
    g0 = d["viewer"]
    own = {_key(d["rules"], t["color"], t["value"]) for t in d["lines"][g0]}
    rev = {_key(d["rules"], t["color"], t["value"]) for line in d["lines"] for t in line if t.get("revealed")}
    out = []
    for dd in range(1, rules.P):
        j = (g0 + dd) % rules.P
        line = d["lines"][j]
        if all(t.get("revealed") for t in line):
            continue
        for pos, t in enumerate(line):
            if t.get("revealed"):
                continue
            c = 0 if t["color"] == "B" else 1
            for v in rules.T:
                if (v & 1) == c and v not in own and v not in rev:
                    out.append((j << 24) | (pos << 16) | v)
    if rules.cons and d.get("correct_this_turn", 0) >= 1:
        out.append(STOP)
    return out


def exact(d, code):
    """p_w(code) for every seat w (tuple of Fractions)."""
    rules, dets = determinizations(d)
    assert dets, "inconsistent observation"
    value = make_value(rules)
    total = [Fraction(0)] * rules.P
    for st in dets:
        st2, step = apply(rules, st, code)
        v = value(st2, step)
        for w in range(rules.P):
            total[w] += Fraction(1, len(dets)) * v[w]
    return tuple(total)


def n_det(d):
    return len(determinizations(d)[1])


# ---------------------------------------------------------------- tiny positions (own generator)

def observe(rules, state, viewer, P):
    lines, rev, pool, g, pend, corr = state
    out = []
    R = rules.R
    for p in range(P):
        ln = []
        for k in materialise(lines[p]):
            r = k in rev
            v = "J" if rules.joker(k) else k >> 1
            if p != viewer and not r:
                v = None
            ln.append({"color": "B" if (k & 1) == 0 else "W", "value": v, "revealed": r})
        out.append(ln)
    pending = -1
    if pend is not None:
        pending = materialise(lines[viewer]).index(pend)
    return {"rules": {"players": P, "ranks": R, "jokers": rules.jok, "consecutive": rules.cons},
            "viewer": viewer, "lines": out, "pool_size": len(pool), "pending": pending,
            "correct_this_turn": corr}


def tiny_position(P, R, jok, cons, per, seed, max_decisions):
    """Deal `per` tiles each (dealt jokers leftmost), seat 0 draws,
    then up to `max_decisions` uniform random decisions (own RNG); returns the
    observation of the mover at AwaitGuess, or None if the game ended."""
    rules = Rules({"players": P, "ranks": R, "jokers": jok, "consecutive": cons})
    rng = random.Random(seed)
    T = list(rules.T)
    rng.shuffle(T)
    lines = []
    for p in range(P):
        hand = T[p * per:(p + 1) * per]
        js = sorted(k for k in hand if rules.joker(k))
        ns = sorted(k for k in hand if not rules.joker(k))
        lines.append((tuple(ns), tuple((k, 0) for k in js)))
    pool = tuple(sorted(T[P * per:]))
    # seat 0's first draw: the turn start of seat P-1's "previous turn"
    state = (tuple(lines), frozenset(), pool, P - 1, None, 0)
    opts = turn_starts(rules, state)
    state = opts[rng.randrange(len(opts))][1] if pool else (state[0], state[1], pool, 0, None, 0)
    for _ in range(rng.randrange(max_decisions + 1)):
        L = legal(rules, state)
        choices = L + ([STOP] if rules.cons and state[5] >= 1 else [])
        st, step = apply(rules, state, choices[rng.randrange(len(choices))])
        if step == "FINISH":
            return None
        if step == "END_TURN":
            opts = turn_starts(rules, st)
            st = opts[rng.randrange(len(opts))][1]
        state = st
    return observe(rules, state, state[3], P)
