"""ORACLE-side analysis (test infrastructure only): the lockstep SIMT model of
SPEC:377-437 (simt-sim), used for SURVEY §8(f) N3 -- the turn-level
divergence the paper blames for its GPU losses ("threads that are already
finished should wait until the thread with the most turns ends").

Lane lengths come from the oracle's playouts (iterations = 1 start + the
decision steps), so the model predicts the naive thread-per-playout kernel's
warp efficiency from the playout-length distribution alone; ncu's measured
smsp__thread_inst_executed_per_inst_executed / 32 is below it by the
intra-step divergence the model ignores.
"""

from . import playout as oracle_playout


def simulate_warp(steps, width):
    """Active-lane count per lockstep cycle (SPEC simulate_warp)."""
    if len(steps) != width:
        raise ValueError("width mismatch")
    return [sum(1 for s in steps if s > t) for t in range(max(steps))]


def simd_efficiency(masks, width):
    """sum(active) / (width * cycles) (SPEC simd_efficiency)."""
    return sum(masks) / (width * len(masks))


def playout_iterations(obs_json, code, seed, node, s0, s1):
    """Kernel iterations (1 start + decisions) of playouts s0..s1-1 of one action."""
    return [1 + oracle_playout(obs_json, code, seed, node, s)[1] for s in range(s0, s1)]


def naive_kernel_efficiency(obs_json, codes, seed, sims_per_action, width=32):
    """Predicted turn-level warp efficiency of the grid-stride naive kernel:
    a warp executes `width` consecutive work items (consecutive sims of one
    action) in lockstep, so each round costs max(lengths) cycles."""
    active = cycles = 0
    for c in codes:
        lens = playout_iterations(obs_json, c, seed, 0, 0, sims_per_action)
        for i in range(0, len(lens) - width + 1, width):
            m = simulate_warp(lens[i:i + width], width)
            active += sum(m)
            cycles += width * len(m)
    return active / cycles
