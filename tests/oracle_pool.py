"""Test helper: run the C++ oracle over disjoint sim sub-ranges in worker
processes and sum the histograms (the all-core oracle of SURVEY §8(d); the sum
over a split equals the unsplit run because playouts are keyed by sim index)."""

import os
from concurrent.futures import ProcessPoolExecutor

_POOL = None


def _work(args):
    import oracle
    d, codes, seed, node, s0, s1 = args
    return oracle.rollout(d, codes, seed, node, s0, s1)


def pool():
    global _POOL
    if _POOL is None:
        import multiprocessing as mp
        _POOL = ProcessPoolExecutor(max_workers=max(1, min(os.cpu_count() or 1, 64)),
                                    mp_context=mp.get_context("spawn"))
    return _POOL


def oracle_hist(d, codes, seed, node, s0, s1, chunks=None):
    n = s1 - s0
    chunks = chunks or max(1, min(n, (os.cpu_count() or 1) * 2))
    bounds = [s0 + (n * i) // chunks for i in range(chunks + 1)]
    jobs = [(d, list(codes), seed, node, bounds[i], bounds[i + 1]) for i in range(chunks) if bounds[i] < bounds[i + 1]]
    P = d["rules"]["players"]
    tot = [[0] * P for _ in codes]
    for h in pool().map(_work, jobs):
        for a in range(len(codes)):
            for w in range(P):
                tot[a][w] += h[a][w]
    return tot
