"""Self-play driver (BASELINE.json configs[2], C3): a referee holds the true
game and asks the player to move for its MCTS decision
(dvc_mcts_search over the GPU rollout batches), from its own observation only.

The referee is a small list-based rules engine (§II-A; the
readings of DESIGN.md §R) with its own seeded RNG for the deal, the draws and
the placement of drawn jokers; it is host bookkeeping, not the hot path.
Protocol (shared by the oracle's self-play for parity):
  deal:  T = [0, |T|); random.Random(seed).shuffle(T); seat p gets
         T[p*per:(p+1)*per]; a line = its jokers (JB, JW) then numbered keys
         ascending; the pool is the rest, sorted;
  draw:  idx = rng.randrange(len(pool)) of the sorted pool; a drawn joker goes
         to gap rng.randrange(len(line) + 1); a numbered key before the first
         larger numbered tile;
  turn:  seat 0 draws first; after a wrong guess or STOP the next alive seat
         draws; the search seed of decision i is seed * 1000003 + i.
"""

import random

STOP = 0xFFFFFFFF


class Referee:
    def __init__(self, players, ranks, jokers, consecutive, per, seed):
        self.P, self.R, self.jokers, self.cons = players, ranks, jokers, consecutive
        self.rng = random.Random(seed)
        nT = 2 * ranks + (2 if jokers else 0)
        T = list(range(nT))
        self.rng.shuffle(T)
        self.lines = []
        for p in range(players):
            hand = T[p * per:(p + 1) * per]
            jk = sorted(k for k in hand if k >= 2 * ranks)
            num = sorted(k for k in hand if k < 2 * ranks)
            self.lines.append([[k, False] for k in jk + num])
        self.pool = sorted(T[players * per:])
        self.g = 0
        self.pend = None
        self.corr = 0

    def is_joker(self, k):
        return k >= 2 * self.R

    def alive(self, p):
        return any(not r for _, r in self.lines[p])

    def over(self):
        return sum(1 for p in range(self.P) if self.alive(p)) <= 1

    def winner(self):
        return [p for p in range(self.P) if self.alive(p)][0]

    def draw(self):
        self.pend, self.corr = None, 0
        if not self.pool:
            return
        t = self.pool.pop(self.rng.randrange(len(self.pool)))
        ln = self.lines[self.g]
        if self.is_joker(t):
            ln.insert(self.rng.randrange(len(ln) + 1), [t, False])
        else:
            i = len(ln)
            for idx, (k, _) in enumerate(ln):
                if not self.is_joker(k) and k > t:
                    i = idx
                    break
            ln.insert(i, [t, False])
        self.pend = t

    def next_turn(self):
        for d in range(1, self.P + 1):
            p = (self.g + d) % self.P
            if self.alive(p):
                self.g = p
                break
        self.draw()

    def observation(self):
        """The mover's view as fixture JSON (SPEC:191 tile shape + extras)."""
        v = self.g
        lines = []
        for p, ln in enumerate(self.lines):
            out = []
            for k, r in ln:
                val = "J" if self.is_joker(k) else k >> 1
                out.append({"color": "B" if (k & 1) == 0 else "W",
                            "value": val if (p == v or r) else None, "revealed": bool(r)})
            lines.append(out)
        pending = -1
        if self.pend is not None:
            pending = [k for k, _ in self.lines[v]].index(self.pend)
        return {"rules": {"players": self.P, "ranks": self.R, "jokers": self.jokers, "consecutive": self.cons},
                "viewer": v, "lines": lines, "pool_size": len(self.pool), "pending": pending,
                "correct_this_turn": self.corr}

    def apply(self, code):
        """Returns (outcome, correct): outcome in FINISH / DECIDE / END_TURN."""
        if code == STOP:
            return "END_TURN", False
        j, pos, v = code >> 24, (code >> 16) & 0xFF, code & 0xFFFF
        if self.lines[j][pos][0] == v:
            self.lines[j][pos][1] = True
            self.corr += 1
            if self.over():
                return "FINISH", True
            return ("DECIDE" if self.cons else "END_TURN"), True
        ln = self.lines[self.g]
        idx = None
        if self.pend is not None:
            for i, (k, r) in enumerate(ln):
                if k == self.pend and not r:
                    idx = i
        if idx is None:
            idx = next(i for i, (_, r) in enumerate(ln) if not r)
        ln[idx][1] = True
        return ("FINISH" if self.over() else "END_TURN"), False


def play_game(seed, players=2, ranks=12, jokers=1, consecutive=1, per=4, expansions=64, sims_per_child=1024,
              max_depth=4, flat=1, search=None, max_decisions=500):
    """One self-play game; every decision is dvc_mcts_search from the mover's
    observation (or `search(obs_json, seed) -> code` if given).  Returns
    {"winner", "moves": [(mover, code, correct)], "decisions"}."""
    if search is None:
        from . import dvc

        def search(obs, s):
            st = dvc.encode(obs)
            best, _ = dvc.mcts_search(st, expansions, sims_per_child, s, max_depth=max_depth, flat=flat)
            return best
    ref = Referee(players, ranks, jokers, consecutive, per, seed)
    ref.draw()
    moves = []
    for i in range(max_decisions):
        obs = ref.observation()
        code = search(obs, seed * 1000003 + i)
        mover = ref.g
        out, correct = ref.apply(code)
        moves.append((mover, code, correct))
        if out == "FINISH":
            return {"winner": ref.winner(), "moves": moves, "decisions": len(moves)}
        if out == "END_TURN":
            ref.next_turn()
    raise RuntimeError("game did not finish within %d decisions" % max_decisions)


def play_games(seeds, threads=8, **kw):
    """Several self-play games at once, one host thread each: every thread's
    blocking searches run on its own CUDA stream (the library keeps a stream
    per host thread), so the small per-decision batches of different games
    overlap on the GPU.  Results are identical to playing the games one by
    one (every decision is a pure function of its inputs)."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda s: play_game(s, **kw), seeds))
