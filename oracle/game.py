"""ORACLE (test infrastructure only) -- plain, slow, list-based Da Vinci Code rules,
determinization sampler and Philox-driven playout, written from the paper in the
order of DESIGN.md §R1-§R6 (= SURVEY.md §8(c.1)-(c.6)).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may
import anything under `oracle/`; the product path never does, and this module
shares no code with `paper_2403_10720_b200/`.

Passages followed:
  * rules: PAPER:102-106 (§II-A, Fig. 1) -- draw and insert in ascending order,
    guess an opponent tile, a correct guess reveals it and grants another guess,
    a wrong guess reveals the guesser's newly drawn tile, last gambler standing;
  * random playout: PAPER:114 ("selecting decision at random");
  * determinization: PAPER:143 ("A set of these plausible numbers is randomly
    selected for each simulation");
  * stop-after-a-correct-guess variant: PAPER:153 (rule flag consecutive=0);
  * binary outcome / merge-by-sum: PAPER:180, 183, 186;
  * readings where the paper is silent: DESIGN.md §R7 (= SURVEY.md §8(c.7)).

Representation (deliberately naive): a line is a Python list of [key, revealed]
in left-to-right order; the pool is a sorted list of keys.  Keys: numbered tile
(rank r, colour c) -> 2r+c; jokers JB = 2R, JW = 2R+1; colour(key) = key & 1.
"""

from . import philox as px

STOP = 0xFFFFFFFF
BIG = 1 << 30      # "no revealed numbered tile on this side" (order_bounds)
NONE = -1


# ----------------------------------------------------------------- encodings (§R1)

class Rules:
    def __init__(self, players, ranks=12, jokers=0, consecutive=1):
        self.P = int(players)
        self.R = int(ranks)
        self.jokers = int(jokers)
        self.consecutive = int(consecutive)
        if self.P not in (2, 3, 4) or not (1 <= self.R <= 12) \
                or self.jokers not in (0, 1) or self.consecutive not in (0, 1):
            raise ValueError("config")

    @property
    def JB(self):
        return 2 * self.R

    @property
    def JW(self):
        return 2 * self.R + 1

    def tiles(self):
        """The tile set T in ascending key order."""
        n = 2 * self.R + (2 if self.jokers else 0)
        return list(range(n))

    def is_joker(self, k):
        return k >= 2 * self.R

    def key_of(self, color, value):
        c = 0 if color in ("B", 0) else 1
        if value == "J":
            return 2 * self.R + c
        return 2 * int(value) + c


def colour(k):
    return k & 1


def action_code(target, pos, value_key):
    return (target << 24) | (pos << 16) | value_key


def decode_action(code):
    return code >> 24, (code >> 16) & 0xFF, code & 0xFFFF


# ----------------------------------------------------------------- observation

class Observation:
    """The viewer's information set at AwaitGuess (SPEC:63-68 shape plus the
    `pending` / `correct_this_turn` extras of SURVEY.md §8(b)).

    lines[p] = list of (colour, key or None, revealed); the viewer's own line is
    fully valued, an opponent's hidden tile has key None.
    """

    def __init__(self, rules, viewer, lines, pool_size, pending, correct_this_turn):
        self.rules = rules
        self.viewer = viewer
        self.lines = lines
        self.pool_size = pool_size
        self.pending = pending
        self.corr = correct_this_turn

    @staticmethod
    def from_json(d):
        r = d["rules"]
        rules = Rules(r["players"], r.get("ranks", 12), r.get("jokers", 0), r.get("consecutive", 1))
        lines = []
        for line in d["lines"]:
            out = []
            for t in line:
                c = 0 if t["color"] == "B" else 1
                v = t.get("value")
                k = None if v is None else rules.key_of(c, v)
                out.append((c, k, bool(t.get("revealed", False))))
            lines.append(out)
        return Observation(rules, int(d["viewer"]), lines, int(d["pool_size"]),
                           int(d.get("pending", -1)), int(d.get("correct_this_turn", 0)))


# ----------------------------------------------------------------- game state

class Game:
    """Full-information state inside one playout (§R5)."""

    def __init__(self, rules, lines, pool, g, pend, corr):
        self.rules = rules
        self.lines = lines      # list (per seat) of list of [key, revealed]
        self.pool = pool        # sorted list of keys
        self.g = g              # mover
        self.pend = pend        # this turn's drawn key, or NONE
        self.corr = corr        # correct guesses this turn

    def copy(self):
        return Game(self.rules, [[list(t) for t in ln] for ln in self.lines],
                    list(self.pool), self.g, self.pend, self.corr)

    def key_state(self):
        return (tuple(tuple((k, r) for k, r in ln) for ln in self.lines),
                tuple(self.pool), self.g, self.pend, self.corr)

    # --- predicates
    def hand(self, p):
        return {k for k, _ in self.lines[p]}

    def revealed_keys(self):
        return {k for ln in self.lines for k, r in ln if r}

    def alive(self, p):
        return any(not r for _, r in self.lines[p])

    def n_alive(self):
        return sum(1 for p in range(self.rules.P) if self.alive(p))

    def over(self):
        return self.n_alive() <= 1

    def winner(self):
        alive = [p for p in range(self.rules.P) if self.alive(p)]
        assert len(alive) == 1
        return alive[0]

    # --- line operations (§R2)
    def insert_numbered(self, p, t):
        """A numbered key goes immediately before the first numbered tile with a
        larger key (so it lands right of any joker in its gap)."""
        ln = self.lines[p]
        i = len(ln)
        for idx, (k, _) in enumerate(ln):
            if not self.rules.is_joker(k) and k > t:
                i = idx
                break
        ln.insert(i, [t, False])

    def insert_joker(self, p, t, gap):
        """A drawn joker goes into gap `gap` in 0..len(line)."""
        self.lines[p].insert(gap, [t, False])

    def leftmost_hidden(self, p):
        for idx, (_, r) in enumerate(self.lines[p]):
            if not r:
                return idx
        raise AssertionError("no hidden tile")

    # --- legal guesses (§R5 LEGAL)
    def legal(self, informed=False):
        """LEGAL(g) (§R5); informed: the order-aware policy list (§R10) -- a
        numbered value must lie strictly between the nearest revealed numbered
        tiles left and right of the slot; a joker value is always kept."""
        P, g = self.rules.P, self.g
        own = self.hand(g)
        rev = self.revealed_keys()
        out = []
        for d in range(1, P):
            j = (g + d) % P
            if not self.alive(j):
                continue
            for pos, (k, r) in enumerate(self.lines[j]):
                if r:
                    continue
                c = colour(k)
                if informed:
                    lo, hi = self.order_bounds(j, pos)
                for v in self.rules.tiles():
                    if colour(v) != c:
                        continue
                    if v in own or v in rev:
                        continue
                    if informed and not self.rules.is_joker(v) and not (lo < v < hi):
                        continue
                    out.append(action_code(j, pos, v))
        return out

    def order_bounds(self, j, pos):
        """(lo, hi): keys of the nearest revealed numbered tiles left and right
        of position pos in line j, -1 / BIG when there is none (§R10).  The
        revealed numbered keys increase along a line, so the last one on the
        left is the largest and the first one on the right the smallest."""
        lo, hi = -1, BIG
        for p, (k, r) in enumerate(self.lines[j]):
            if not r or self.rules.is_joker(k):
                continue
            if p < pos:
                lo = k
            elif p > pos and hi == BIG:
                hi = k
        return lo, hi

    def n_choices(self, legal):
        stop = 1 if (self.rules.consecutive and self.corr >= 1) else 0
        return len(legal) + stop

    # --- apply a decision (§R5 APPLY). Returns "FINISH" | "DECIDE" | "END_TURN".
    def apply(self, code):
        if code == STOP:
            return "END_TURN"
        j, pos, v = decode_action(code)
        t = self.lines[j][pos][0]
        if t == v:
            self.lines[j][pos][1] = True
            self.corr += 1
            if self.over():
                return "FINISH"
            return "DECIDE" if self.rules.consecutive else "END_TURN"
        g = self.g
        ln = self.lines[g]
        idx = None
        if self.pend != NONE:
            for i2, (k, r) in enumerate(ln):
                if k == self.pend and not r:
                    idx = i2
        if idx is None:
            idx = self.leftmost_hidden(g)
        ln[idx][1] = True
        return "FINISH" if self.over() else "END_TURN"

    def next_mover(self):
        P = self.rules.P
        for d in range(1, P + 1):
            p = (self.g + d) % P
            if self.alive(p):
                return p
        raise AssertionError

    def start_turn(self, w, gap_word=None):
        """END_TURN handling: next alive player, draw with word w = b0 (§R3):
        pool index choose(|Q|, w); a drawn joker's gap from the remainder.
        (gap_word: the fixture generator's own second word, not the contract.)"""
        self.g = self.next_mover()
        self.pend = NONE
        self.corr = 0
        if self.pool:
            q = len(self.pool)
            t = self.pool.pop(px.choose(q, w))
            if self.rules.is_joker(t):
                gw = px.remainder(q, w) if gap_word is None else gap_word
                gap = px.choose(len(self.lines[self.g]) + 1, gw)
                self.insert_joker(self.g, t, gap)
            else:
                self.insert_numbered(self.g, t)
            self.pend = t


def root_legal(obs, informed=False):
    """LEGAL(g0) under the viewer's information, plus STOP when allowed (§R5);
    informed: the order-aware list (§R10)."""
    g = _public_game(obs)
    codes = g.legal(informed)
    if obs.rules.consecutive and obs.corr >= 1:
        codes.append(STOP)
    return codes


def _public_game(obs):
    """A Game whose opponent hidden keys are placeholders; only good for LEGAL at
    the root (which never reads a hidden key's value, only its colour)."""
    R = obs.rules
    lines = []
    for ln in obs.lines:
        out = []
        for c, k, r in ln:
            # placeholder for a hidden tile: a key of the right colour that is
            # outside T, so it is never "in own hand" nor "revealed".
            out.append([k if k is not None else 1000 + c, r])
        lines.append(out)
    return Game(R, lines, [], obs.viewer, NONE, obs.corr)


# ----------------------------------------------------------------- determinization (§R4)

class DetSpace:
    """Det(O): the consistent assignments of hidden opponent slots, in the
    canonical lexicographic order of delta = (o_JB, o_JW, d_0, ..., d_{m-1}).

    Follows SURVEY.md §8(c.4) "Reference algorithm" step by step:
      1. joint joker options (o_JB major, o_JW minor); chains per opponent;
      2. N(i, q) by memoised recursion over the numbered keys u_0 < ... of U;
      3. N = sum over joint options;
      4. unrank by walking joint options then keys, options [pool, d=1..P-1].
    """

    def __init__(self, obs):
        self.obs = obs
        R = obs.rules
        P, g0 = R.P, obs.viewer
        self.P, self.g0 = P, g0
        known = {k for c, k, r in obs.lines[g0]}
        for p in range(P):
            if p == g0:
                continue
            for c, k, r in obs.lines[p]:
                if r:
                    known.add(k)
        self.U = [k for k in R.tiles() if k not in known]
        self.numbered_U = [k for k in self.U if not R.is_joker(k)]
        # hidden slots in HS order: seat offset d = 1..P-1, then line index
        self.HS = []
        for d in range(1, P):
            j = (g0 + d) % P
            for idx, (c, k, r) in enumerate(obs.lines[j]):
                if not r:
                    self.HS.append((d, idx, c))
        # joker options: 0 = pool, 1 + t = t-th HS slot of the joker's colour
        self.joker_dims = []   # list of (joker key, [option -> HS index or None])
        if R.jokers:
            for J in (R.JB, R.JW):
                if J in self.U:
                    slots = [h for h, (d, idx, c) in enumerate(self.HS) if c == colour(J)]
                    self.joker_dims.append((J, [None] + slots))
        self.options = self._joint_options()
        self.counts = [self._count_option(opt) for opt in self.options]
        self.N = sum(self.counts)

    def _joint_options(self):
        opts = [()]
        for J, choices in self.joker_dims:
            opts = [o + (h,) for o in opts for h in choices]
        # drop infeasible joint options (both jokers in one slot cannot happen:
        # the jokers have different colours)
        return opts

    def _chains(self, opt):
        """Per opponent (offset order): remaining hidden slots in line order with
        (colour, lo, hi); lo/hi = key of nearest revealed numbered tile to the
        left/right (-1 / 2R if none).  Jokers are ignored for order."""
        R = self.obs.rules
        taken = {h for h in opt if h is not None}
        chains = []
        for d in range(1, self.P):
            j = (self.g0 + d) % self.P
            line = self.obs.lines[j]
            ch = []
            for h, (dd, idx, c) in enumerate(self.HS):
                if dd != d or h in taken:
                    continue
                lo, hi = -1, 2 * R.R
                for i2 in range(idx - 1, -1, -1):
                    c2, k2, r2 = line[i2]
                    if r2 and not R.is_joker(k2):
                        lo = k2
                        break
                for i2 in range(idx + 1, len(line)):
                    c2, k2, r2 = line[i2]
                    if r2 and not R.is_joker(k2):
                        hi = k2
                        break
                ch.append((c, lo, hi))
            chains.append(ch)
        return chains

    @staticmethod
    def _fits(slot, u):
        c, lo, hi = slot
        return colour(u) == c and lo < u < hi

    def _count_option(self, opt):
        chains = self._chains(opt)
        m = len(self.numbered_U)
        memo = {}

        def N(i, q):
            if (i, q) in memo:
                return memo[(i, q)]
            if i == m:
                v = 1 if all(q[j] == len(chains[j]) for j in range(len(chains))) else 0
            else:
                u = self.numbered_U[i]
                v = N(i + 1, q)  # u goes to the pool
                for j in range(len(chains)):
                    if q[j] < len(chains[j]) and self._fits(chains[j][q[j]], u):
                        q2 = q[:j] + (q[j] + 1,) + q[j + 1:]
                        v += N(i + 1, q2)
            memo[(i, q)] = v
            return v

        self._last_memo = (chains, N)
        return N(0, tuple(0 for _ in chains))

    def unrank(self, rho):
        """The rho-th element of Det(O): returns dict HS-index -> key."""
        assert 0 <= rho < self.N
        for opt, cnt in zip(self.options, self.counts):
            if rho >= cnt:
                rho -= cnt
                continue
            assign = {}
            for (J, _), h in zip(self.joker_dims, opt):
                if h is not None:
                    assign[h] = J
            self._count_option(opt)  # rebuild the memo for this option
            chains, N = self._last_memo
            # map chain positions back to HS indices
            taken = {h for h in opt if h is not None}
            chain_hs = []
            for d in range(1, self.P):
                chain_hs.append([h for h, (dd, idx, c) in enumerate(self.HS)
                                 if dd == d and h not in taken])
            q = tuple(0 for _ in chains)
            for i, u in enumerate(self.numbered_U):
                w = N(i + 1, q)                 # option: pool
                if rho < w:
                    continue
                rho -= w
                placed = False
                for j in range(len(chains)):     # options d = 1..P-1
                    if q[j] < len(chains[j]) and self._fits(chains[j][q[j]], u):
                        q2 = q[:j] + (q[j] + 1,) + q[j + 1:]
                        w = N(i + 1, q2)
                        if rho < w:
                            assign[chain_hs[j][q[j]]] = u
                            q = q2
                            placed = True
                            break
                        rho -= w
                assert placed
            assert rho == 0 and all(q[j] == len(chains[j]) for j in range(len(chains)))
            return assign
        raise AssertionError("rho out of range")

    def game(self, assign):
        """The determinized full state at the root (viewer to move)."""
        obs = self.obs
        lines = []
        for p, ln in enumerate(obs.lines):
            out = []
            for idx, (c, k, r) in enumerate(ln):
                out.append([k, r])
            lines.append(out)
        for h, key in assign.items():
            d, idx, c = self.HS[h]
            j = (self.g0 + d) % self.P
            lines[j][idx][0] = key
        used = set(assign.values())
        pool = sorted(k for k in self.U if k not in used)
        assert len(pool) == obs.pool_size
        pend = NONE
        if obs.pending >= 0:
            pend = obs.lines[self.g0][obs.pending][1]
        return Game(obs.rules, lines, pool, self.g0, pend, obs.corr)


# ----------------------------------------------------------------- playout (§R5)

def playout(space, code, seed, node_id, s, trace=None, crn=False, informed=False, rho=None):
    """One playout: determinize with block D, apply the root action, then play
    uniformly random decisions with one Philox2x32 block per decision step
    (b0: draw, b1: decision; §R3).  rho: play determinization rho of Det(O)
    instead of sampling one (the "md" ablation, §R11).
    Returns the winner seat.  crn: D is keyed by CRN_WORD instead of the code
    (common determinizations across actions); informed: every
    decision is uniform over the order-aware list (§R10) instead of LEGAL."""
    if rho is None:
        D = px.det_block(seed, node_id, px.CRN_WORD if crn else code, s)
        rho = px.rank64(space.N, D[0], D[1])
    # else: the "md" ablation's fixed determinization
    game = space.game(space.unrank(rho))
    step = game.apply(code)
    k = 0
    while True:
        if step == "FINISH":
            w = game.winner()
            if trace is not None:
                trace.append(("winner", w))
            return w
        B = px.step_block(seed, node_id, code, s, k)
        if step == "END_TURN":
            game.start_turn(B[0])
        L = game.legal(informed)
        n = game.n_choices(L)
        i = px.choose(n, B[1])
        k += 1
        a = STOP if i == len(L) else L[i]
        if trace is not None:
            trace.append((game.g, a))
        step = game.apply(a)


VOID = "VOID"


def playout_path(space, path, code, seed, node_id, s, trace=None):
    """Deep-tree playout: the viewer's forced actions
    F = path + [code] -- F[0] at the root, F[i] at the viewer's i-th later
    decision -- then uniform random play.  Philox keyed by the batch action
    `code`.  Returns the winner seat, or VOID when a forced action is not in
    LEGAL (+ STOP when allowed) or the game ends before all of F is applied."""
    if not path:
        return playout(space, code, seed, node_id, s, trace)
    F = list(path) + [code]
    viewer = space.g0
    D = px.det_block(seed, node_id, code, s)
    rho = px.rank64(space.N, D[0], D[1])
    game = space.game(space.unrank(rho))
    step = game.apply(F[0])
    fi = 1
    k = 0
    while True:
        if step == "FINISH":
            return VOID if fi < len(F) else game.winner()
        B = px.step_block(seed, node_id, code, s, k)
        if step == "END_TURN":
            game.start_turn(B[0])
        L = game.legal()
        n = game.n_choices(L)
        if fi < len(F) and game.g == viewer:
            a = F[fi]
            fi += 1
            allowed = L + ([STOP] if n > len(L) else [])
            if a not in allowed:
                return VOID
        else:
            i = px.choose(n, B[1])
            a = STOP if i == len(L) else L[i]
        k += 1
        if trace is not None:
            trace.append((game.g, a))
        step = game.apply(a)


def check_action(obs, code):
    if code not in root_legal(obs):
        raise ValueError("illegal action %08x" % code)


def rollout_fixed(obs, codes, rhos, seed, node_id, s0, s1):
    """The "md" ablation batch (§R11): hist[i][w] for child (rhos[i], codes[i])."""
    space = DetSpace(obs)
    if space.N == 0:
        raise ValueError("inconsistent")
    for c, r in zip(codes, rhos):
        check_action(obs, c)
        if not 0 <= r < space.N:
            raise ValueError("rho out of range")
    hist = [[0] * obs.rules.P for _ in codes]
    for ai, (c, r) in enumerate(zip(codes, rhos)):
        for s in range(s0, s1):
            hist[ai][playout(space, c, seed, node_id, s, rho=r)] += 1
    return hist


def rollout(obs, codes, seed, node_id, s0, s1, crn=False, informed=False):
    """hist[a][w] over sims s in [s0, s1) (§R6)."""
    space = DetSpace(obs)
    if space.N == 0:
        raise ValueError("inconsistent")
    for c in codes:
        check_action(obs, c)
    hist = [[0] * obs.rules.P for _ in codes]
    for ai, c in enumerate(codes):
        for s in range(s0, s1):
            hist[ai][playout(space, c, seed, node_id, s, crn=crn, informed=informed)] += 1
    return hist
