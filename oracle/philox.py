"""ORACLE (test infrastructure only) -- the random-number contract of DESIGN.md §R3.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may
import anything under `oracle/`.  The product path (paper_2403_10720_b200/) never
does.

The paper is silent on the RNG ("selecting decision at random",
PAPER:143 "randomly selected for each simulation"); BASELINE.json north_star
fixes "a counter-based Philox keyed by (node, action, sim index)".  This file is
the plain definition: Philox2x32-10 (Salmon, Moraes, Dror, Shaw, SC'11,
"Parallel random numbers: as easy as 1, 2, 3"; Random123's `philox2x32`), the
stream key and counter layout of §R3, and the two integer maps `choose` and
`rank64`.

Pins (tests/test_oracle_philox.py): the Random123 known-answer vectors, the
libcudacxx `cuda::std::philox_engine` (C++26 std::philox_engine) instantiated
as Philox2x32-10, exhaustive bucket sizes of `choose` for small n, rank64
boundaries, the counter packing.
"""

MASK32 = 0xFFFFFFFF
PHILOX2_M = 0xD256D193
PHILOX2_W = 0x9E3779B9

DET_STEP = 63          # step field t of the determinization block D (§R3)
MAX_STEP = 62          # decision steps t = 0..62 after the root action
# Common-random-numbers variant: the
# determinization block takes this word in place of the action code, so every
# action of a batch sees the same hidden-tile assignment for a given sim index.
# 0xFFFFFFFE is no action code (targets are <= 3, STOP is 0xFFFFFFFF).
CRN_WORD = 0xFFFFFFFE
STOP_CODE = 0xFFFFFFFF


def philox2x32_10(ctr, key):
    """Philox2x32 with 10 rounds.  ctr: 2 x u32, key: u32 -> 2 x u32.

    One round: (hi, lo) = M * c0;  c' = (hi ^ k ^ c1, lo);
    the key is bumped by W between rounds (SC'11, §4 "Philox").
    """
    c0, c1 = (int(x) & MASK32 for x in ctr)
    k = int(key) & MASK32
    for r in range(10):
        if r > 0:
            k = (k + PHILOX2_W) & MASK32
        p = PHILOX2_M * c0
        hi, lo = p >> 32, p & MASK32
        c0, c1 = hi ^ k ^ c1, lo
    return (c0, c1)


def stream_key(seed, node_id):
    """K = word 0 of Philox2x32-10(ctr=(lo32(seed), hi32(seed)), key=node)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return philox2x32_10((seed & MASK32, seed >> 32), int(node_id) & MASK32)[0]


def code12(code):
    """12-bit image of an action code (§R3): target<<10 | position<<5 | value;
    STOP -> 0xFFF, CRN_WORD -> 0xFFE (position 31 never occurs: lines <= 26)."""
    code = int(code) & MASK32
    if code == STOP_CODE:
        return 0xFFF
    if code == CRN_WORD:
        return 0xFFE
    target, pos, val = code >> 24, (code >> 16) & 0xFF, code & 0xFFFF
    assert target <= 3 and pos <= 25 and val <= 27, "not an action code: %08x" % code
    return (target << 10) | (pos << 5) | val


def counter(s, t, code, node_id):
    """(c0, c1) = (s, t | code12 << 6 | (node mod 2^14) << 18)."""
    assert 0 <= t <= DET_STEP
    return (int(s) & MASK32, t | (code12(code) << 6) | ((int(node_id) & 0x3FFF) << 18))


def det_block(seed, node_id, code, s):
    """Determinization block D (step field 63): 2 words (d0, d1)."""
    return philox2x32_10(counter(s, DET_STEP, code, node_id), stream_key(seed, node_id))


def step_block(seed, node_id, code, s, t):
    """Decision-step block B_t, t = 0..62: 2 words (b0, b1)."""
    assert 0 <= t <= MAX_STEP, "more than 63 decisions in one playout"
    return philox2x32_10(counter(s, t, code, node_id), stream_key(seed, node_id))


def choose(n, w):
    """Uniform index in [0, n) from one 32-bit word: floor(w * n / 2^32)."""
    assert 1 <= n < (1 << 32)
    return ((int(w) & MASK32) * n) >> 32


def remainder(n, w):
    """The word left over by choose(n, w): (w * n) mod 2^32 (§R3: the joker
    gap of a drawn joker is choose(len + 1, remainder(|Q|, b0)))."""
    return ((int(w) & MASK32) * n) & MASK32


def rank64(N, w0, w1):
    """Uniform index in [0, N) from two words: floor((w1*2^32 + w0) * N / 2^64)."""
    assert 1 <= N < (1 << 64)
    return ((((int(w1) & MASK32) << 32) | (int(w0) & MASK32)) * N) >> 64
