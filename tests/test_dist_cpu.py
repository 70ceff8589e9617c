"""Multi-rank host logic of the root-parallel merge
on CPU: world_size 2 and 3 over gloo (127.0.0.1).  Each rank takes its
contiguous shard of every action's sim range (dist.shard_range), computes its
histogram with the oracle (the GPU kernel's stand-in on a CPU box; the GPU
path is covered by tests/test_gpu_parity.py's split-range invariance), and
dist.merge_hist sums them; the merged counts must equal the unsplit run."""

import json
import os
import socket

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, path, n, out_dir):
    import torch.distributed as dist
    import oracle
    from paper_2403_10720_b200 import dist as ddist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = json.load(open(path))
    codes = oracle.legal(d)
    s0, s1 = ddist.shard_range(n, rank, world)
    P = d["rules"]["players"]
    local = oracle.rollout(d, codes, 5, 0, s0, s1) if s1 > s0 else [[0] * P for _ in codes]
    h = torch.tensor(local, dtype=torch.int64)
    ddist.merge_hist(h)
    with open(os.path.join(out_dir, "r%d.json" % rank), "w") as f:
        json.dump({"hist": h.tolist(), "range": [s0, s1]}, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 301), (3, 50), (3, 2)])
def test_sharded_merge_equals_unsplit(oracle_lib, tmp_path, world, n):
    import torch.multiprocessing as mp
    path = os.path.join(ROOT, "fixtures", "c2_d3.json")
    mp.spawn(_worker, args=(world, _free_port(), path, n, str(tmp_path)), nprocs=world, join=True)
    d = json.load(open(path))
    codes = oracle_lib.legal(d)
    exp = oracle_lib.rollout(d, codes, 5, 0, 0, n)
    ranges = []
    for r in range(world):
        res = json.load(open(os.path.join(str(tmp_path), "r%d.json" % r)))
        assert res["hist"] == exp            # every rank holds the merged totals
        ranges.append(res["range"])
    # the shards tile [0, n) exactly
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def test_shard_range_properties():
    from paper_2403_10720_b200.dist import shard_range
    for n in (0, 1, 7, 1000003, 1 << 32):
        for world in (1, 2, 3, 8):
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def _search_worker(rank, world, port, out_dir, jobs):
    """dist.mcts_search over gloo with the oracle standing in for the GPU
    batches (a CPU mirror of tests/test_gpu_dist.py): the C++ UCT loop of
    dvc_mcts_search_cb, the sharding and the all_reduce are the product's."""
    import numpy as np
    import torch.distributed as dist
    import oracle
    from paper_2403_10720_b200 import dist as ddist, dvc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    for key, path, (exp_n, n, seed, flat) in jobs:
        d = json.load(open(os.path.join(ROOT, path)))
        st = dvc.encode(d)
        dvc.rollout_batch_ex = lambda s_, codes, sd, node, a, b, crn=False, informed=False: np.array(
            oracle.rollout(d, codes, sd, node, a, b, crn=crn, informed=informed), dtype=np.uint64)

        def path_ex(s_, path_, codes, sd, node, a, b):
            h, v = oracle.rollout_path(d, path_, codes, sd, node, a, b)
            return np.array(h, dtype=np.uint64), np.array(v, dtype=np.uint64)
        dvc.rollout_path_ex = path_ex
        best, stats = ddist.mcts_search(st, exp_n, n, seed, flat=flat)
        res[key] = [best, [list(map(int, t)) for t in stats]]
    with open(os.path.join(out_dir, "r%d.json" % rank), "w") as f:
        json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


def test_replicated_tree_search_world2(oracle_lib, tmp_path):
    """Two ranks run the library's search (UCB1 by ln_series in C++), each
    batch sharded and all-reduced: both ranks end with the oracle search's
    table (flat and depth-capped), i.e. no UCT arithmetic happens in Python."""
    import torch.multiprocessing as mp
    from oracle.search import flat_search, deep_search
    jobs = [("flat", "fixtures/c2_d3.json", (30, 41, 3, 1)), ("deep", "tests/golden/T2c1.json", (12, 17, 4, 0))]
    mp.spawn(_search_worker, args=(2, _free_port(), str(tmp_path), jobs), nprocs=2, join=True)
    ranks = [json.load(open(os.path.join(str(tmp_path), "r%d.json" % r))) for r in range(2)]
    for key, path, (exp_n, n, seed, flat) in jobs:
        d = json.load(open(os.path.join(ROOT, path)))
        bo, so = flat_search(d, exp_n, n, seed) if flat else deep_search(d, exp_n, n, seed)
        assert ranks[0][key] == ranks[1][key] == [bo, [list(t) for t in so]], key
