"""Root-parallel rollouts across GPUs.

The paper's threads each build a mini-tree from the root and the trees are
"amalgamated"; merging root statistics is a sum.  Here every rank
plays the SAME actions on a contiguous slice of every action's sim range,
[floor(r n / G), floor((r+1) n / G)), and one NCCL all_reduce(SUM) over the
int64 histogram merges them.  Because playouts are keyed by sim index
(DESIGN.md §R3), the result is bit-identical for every G.

One process per GPU (torchrun); torch.distributed is plumbing only.
"""

import torch
import torch.distributed as dist

from . import dvc


def shard_range(n, rank, world):
    """Contiguous sim sub-range of rank `rank` out of [0, n)."""
    return (n * rank) // world, (n * (rank + 1)) // world


def merge_hist(hist, group=None):
    """a6: SUM all-reduce of the per-rank int64 winner histograms (NCCL on CUDA
    tensors; any torch.distributed backend for the host-side tests)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist


def rollout_batch_device(state, actions, n_sims, seed, node_id=0, sim_offset=0, group=None, stream=None,
                         crn=False):
    """Sharded rollout; returns the merged int64 [A, P] histogram ON DEVICE
    (every rank holds the same totals after the all_reduce).  crn: common
    determinizations across actions."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    s0, s1 = shard_range(n_sims, rank, world)
    dev = torch.device("cuda", torch.cuda.current_device())
    hist = torch.zeros((len(actions), state.players), dtype=torch.int64, device=dev)
    if s1 > s0:
        dvc.rollout_batch_async(state, actions, seed, node_id, sim_offset + s0, sim_offset + s1, hist,
                                stream=stream, crn=crn)
    return merge_hist(hist, group)


def rollout_batch(state, actions, n_sims, seed, node_id=0, sim_offset=0, group=None, crn=False):
    """As rollout_batch_device, read back to host (numpy-compatible int64 tensor)."""
    return rollout_batch_device(state, actions, n_sims, seed, node_id, sim_offset, group, crn=crn).cpu()


def mcts_search(state, expansions, sims_per_child, seed, c=2 ** 0.5, group=None):
    """Flat root-parallel MCTS on every rank (the tree is replicated: all ranks
    see the same all-reduced counts, so they make the same UCB1 choices and no
    tree is ever broadcast).  Each iteration's batch of the selected child is
    sharded over the ranks' sim ranges (DESIGN.md §R8 / §P).  Same result as
    dvc_mcts_search on one GPU.  Returns (best_code, [(code, visits, wins)])."""
    import math
    codes = state.legal_actions()
    viewer = state.info["viewer"]
    visits = [0] * len(codes)
    wins = [0] * len(codes)
    N = 0
    # root expansion: the unvisited children, in ascending code order, as one
    # leaf-parallel batch (exactly the iterations sequential UCB1 would run)
    k = min(expansions, len(codes))
    order = sorted(range(len(codes)), key=lambda a: codes[a])[:k]
    h = rollout_batch(state, [codes[a] for a in order], sims_per_child, seed, 0, 0, group)
    for i, a in enumerate(order):
        visits[a] = sims_per_child
        wins[a] = int(h[i, viewer])
        N += sims_per_child
    for _ in range(expansions - k):
        best, bv = None, None
        for a in range(len(codes)):
            if visits[a] == 0:
                v = math.inf
            else:
                v = wins[a] / visits[a] + c * math.sqrt(math.log(N) / visits[a])
            if best is None or v > bv or (v == bv and codes[a] < codes[best]):
                best, bv = a, v
        h = rollout_batch(state, [codes[best]], sims_per_child, seed, 0, visits[best], group)
        visits[best] += sims_per_child
        wins[best] += int(h[0, viewer])
        N += sims_per_child
    stats = list(zip(codes, visits, wins))
    best_code = min(stats, key=lambda t: (-t[1], -t[2], t[0]))[0]
    return best_code, stats
