"""GPU: the cross-GPU merge ("amalgamated")
driven through the REAL kernels by several ranks.  A gpurun box has one GPU,
so 2, 3, 4 and 8 ranks (SURVEY §8(c.8) schedule invariance, G in {1,2,4,8})
share it over gloo (dist.merge_hist reduces a host copy); the code path is the one torchrun + NCCL runs on 8 GPUs (shard, launch, SUM
all_reduce), minus the transport.  Checked against the unsplit one-rank run
and the oracle, including n < world (ranks with an empty shard), and the
replicated-tree search (dist.mcts_search: the library's UCT over sharded
batches) against dvc_mcts_search and oracle/search.py."""

import json
import os
import socket

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, jobs):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=180))
    torch.cuda.set_device(0)
    from paper_2403_10720_b200 import dist as ddist, dvc
    res = {}
    for key, kind, path, args in jobs:
        d = json.load(open(os.path.join(ROOT, path)))
        st = dvc.encode(d)
        if kind == "batch":
            n, seed, off = args
            h = ddist.rollout_batch(st, st.legal_actions(), n, seed, 0, off)
            res[key] = h.tolist()
        elif kind == "batch_stream":
            # launched on a side stream: the merge (on the current stream)
            # must be ordered after the kernel
            n, seed, off = args
            side = torch.cuda.Stream()
            h = ddist.rollout_batch_device(st, st.legal_actions(), n, seed, 0, off, stream=side)
            res[key] = h.cpu().tolist()
        else:
            exp_n, n, seed, flat = args
            best, stats = ddist.mcts_search(st, exp_n, n, seed, flat=flat)
            res[key] = [best, [list(map(int, t)) for t in stats]]
    with open(os.path.join(out_dir, "r%d.json" % rank), "w") as f:
        json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


BATCH_JOBS = [("c2_300", "batch", "fixtures/c2_d1.json", (300001, 7, 0)),
              ("c4_small", "batch", "fixtures/c4_d2.json", (2, 3, 0)),        # n < world for world 3
              ("x3_off", "batch", "fixtures/x3_d1.json", (5000, 9, 1 << 20)),
              ("c3_j", "batch", "fixtures/c3_d2.json", (20011, 5, 0)),
              ("c2_side", "batch_stream", "fixtures/c2_d1.json", (1000003, 8, 0))]
SEARCH_JOBS = [("s_flat", "search", "fixtures/c3_d1.json", (96, 257, 21, 1)),
               ("s_deep", "search", "fixtures/c2_d2.json", (40, 129, 5, 0)),
               ("s_x3", "search", "fixtures/x3_d1.json", (60, 65, 2, 1))]


@pytest.fixture(scope="module")
def dvc():
    from paper_2403_10720_b200 import build
    build.build()
    from paper_2403_10720_b200 import dvc as m
    return m


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_multi_rank_merge_on_gpu(dvc, oracle_lib, tmp_path, world):
    import torch.multiprocessing as mp
    jobs = BATCH_JOBS + SEARCH_JOBS
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), jobs), nprocs=world, join=True)
    ranks = [json.load(open(os.path.join(str(tmp_path), "r%d.json" % r))) for r in range(world)]
    from oracle.search import flat_search, deep_search
    for key, kind, path, args in jobs:
        d = json.load(open(os.path.join(ROOT, path)))
        st = dvc.encode(d)
        for r in range(1, world):
            assert ranks[r][key] == ranks[0][key], (key, r)       # every rank holds the merged result
        if kind in ("batch", "batch_stream"):
            n, seed, off = args
            codes = st.legal_actions()
            one = dvc.rollout_batch_ex(st, codes, seed, 0, off, off + n).tolist()
            assert ranks[0][key] == one, key                      # == the unsplit single-rank run
            if n <= 5000:
                assert ranks[0][key] == oracle_lib.rollout(d, codes, seed, 0, off, off + n), key
            elif n <= 400000:                                     # oracle on a strided sample of rows
                for a in range(0, len(codes), 7):
                    sub = oracle_lib.rollout(d, [codes[a]], seed, 0, off, off + n)[0]
                    assert ranks[0][key][a] == sub, (key, a)
        else:
            exp_n, n, seed, flat = args
            best, stats = dvc.mcts_search(st, exp_n, n, seed, flat=flat)
            assert ranks[0][key] == [best, [list(map(int, t)) for t in stats]], key
            if flat:
                bo, so = flat_search(d, exp_n, n, seed)
            else:
                bo, so = deep_search(d, exp_n, n, seed)
            assert ranks[0][key] == [bo, [list(t) for t in so]], key
