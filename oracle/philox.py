"""ORACLE (test infrastructure only) -- the random-number contract of DESIGN.md §R3.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may
import anything under `oracle/`.  The product path (paper_2403_10720_b200/) never
does.

The paper is silent on the RNG ("selecting decision at random",
PAPER:143 "randomly selected for each simulation"); BASELINE.json north_star
fixes "a counter-based Philox keyed by (node, action, sim index)".  This file is
the plain definition: Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11,
"Parallel random numbers: as easy as 1, 2, 3"), the two integer maps `choose`
and `rank64`, and the counter layout of SURVEY.md §8(c.3).

Pins (tests/test_oracle_philox.py): the Random123 known-answer vectors,
exhaustive bucket sizes of `choose` for small n, rank64 boundaries.
"""

MASK32 = 0xFFFFFFFF
PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85

DET_CTR_X = 0xFFFFFFFF  # counter word x of the determinization block (§R3)
# Common-random-numbers variant: the
# determinization block takes this word in place of the action code, so every
# action of a batch sees the same hidden-tile assignment for a given sim index.
# 0xFFFFFFFE is no action code (targets are <= 3, STOP is 0xFFFFFFFF).
CRN_WORD = 0xFFFFFFFE


def philox4x32_10(ctr, key):
    """Philox4x32 with 10 rounds.  ctr: 4 x u32, key: 2 x u32 -> 4 x u32.

    One round: (hi0, lo0) = M0*c0, (hi1, lo1) = M1*c2,
               c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0);
    the key is bumped by (W0, W1) between rounds (SC'11, §4 "Philox").
    """
    c0, c1, c2, c3 = (int(x) & MASK32 for x in ctr)
    k0, k1 = (int(x) & MASK32 for x in key)
    for r in range(10):
        if r > 0:
            k0 = (k0 + PHILOX_W0) & MASK32
            k1 = (k1 + PHILOX_W1) & MASK32
        p0 = PHILOX_M0 * c0
        p1 = PHILOX_M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK32
        hi1, lo1 = p1 >> 32, p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return (c0, c1, c2, c3)


def seed_key(seed):
    """Key = (lo32(seed), hi32(seed)) -- one key for the whole batch (§R3)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return (seed & MASK32, seed >> 32)


def det_block(seed, node_id, code, s):
    """Determinization block D = Philox(ctr=(0xFFFFFFFF, s, code, node_id))."""
    return philox4x32_10((DET_CTR_X, s, code, node_id), seed_key(seed))


def step_block(seed, node_id, code, s, t):
    """Decision-step block B_t = Philox(ctr=(t, s, code, node_id))."""
    return philox4x32_10((t, s, code, node_id), seed_key(seed))


def choose(n, w):
    """Uniform index in [0, n) from one 32-bit word: floor(w * n / 2^32)."""
    assert 1 <= n < (1 << 32)
    return ((int(w) & MASK32) * n) >> 32


def rank64(N, w0, w1):
    """Uniform index in [0, N) from two words: floor((w1*2^32 + w0) * N / 2^64)."""
    assert 1 <= N < (1 << 64)
    return ((((int(w1) & MASK32) << 32) | (int(w0) & MASK32)) * N) >> 64
