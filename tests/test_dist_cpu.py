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
