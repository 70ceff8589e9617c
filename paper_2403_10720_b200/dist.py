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
    """a6: SUM all-reduce of the per-rank int64 winner histograms, in place
    (NCCL on CUDA tensors; a gloo group reduces a host copy of a CUDA tensor,
    which lets several ranks share one GPU in the tests)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if hist.is_cuda and dist.get_backend(group) != "nccl":
            h = hist.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            hist.copy_(h)
        else:
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
    cur = torch.cuda.current_stream(dev)
    if stream is not None:
        stream.wait_stream(cur)          # the kernel adds into hist after its zero fill
    if s1 > s0:
        dvc.rollout_batch_async(state, actions, seed, node_id, sim_offset + s0, sim_offset + s1, hist,
                                stream=stream, crn=crn)
    if stream is not None:
        # the all_reduce (and a gloo host copy) run on torch's current stream:
        # order them after the kernel on the caller's stream
        cur.wait_stream(stream)
    return merge_hist(hist, group)


def rollout_batch(state, actions, n_sims, seed, node_id=0, sim_offset=0, group=None, crn=False):
    """As rollout_batch_device, read back to host (numpy-compatible int64 tensor)."""
    return rollout_batch_device(state, actions, n_sims, seed, node_id, sim_offset, group, crn=crn).cpu()


def sharded_batch(state, group=None):
    """A batch callback for dvc.mcts_search_cb: this rank plays its contiguous
    shard of [sim_begin, sim_end) on its GPU, then one SUM all_reduce of
    (hist, voids) gives every rank the counts of the whole range.
    NCCL groups reduce a CUDA tensor, others (gloo) a CPU tensor."""
    import numpy as np

    def batch(path, actions, seed, node_id, sim_begin, sim_end, flags):
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        a, b = shard_range(sim_end - sim_begin, rank, world)
        a, b = sim_begin + a, sim_begin + b
        P = state.players
        hist = np.zeros((len(actions), P), dtype=np.uint64)
        voids = np.zeros(len(actions), dtype=np.uint64)
        if b > a:
            if path:
                hist, voids = dvc.rollout_path_ex(state, path, actions, seed, node_id, a, b)
            else:
                hist = dvc.rollout_batch_ex(state, actions, seed, node_id, a, b, crn=bool(flags & dvc.FLAG_CRN),
                                            informed=bool(flags & dvc.FLAG_INFORMED))
        t = torch.from_numpy(np.concatenate([hist.reshape(-1), voids]).astype(np.int64))
        if dist.is_initialized() and dist.get_backend(group) == "nccl":
            t = t.cuda()
        merge_hist(t, group)
        t = t.cpu().numpy().astype(np.uint64)
        return t[:len(actions) * P].reshape(len(actions), P), (t[len(actions) * P:] if path else None)

    return batch


def mcts_search(state, expansions, sims_per_child, seed, c=2 ** 0.5, group=None, max_depth=4, flat=1, crn=False,
                informed=False):
    """Root-parallel MCTS (dvc_mcts_search_cb): every rank runs the library's
    search (UCB1 by ln_series, reading #28; flat or depth-capped tree), the
    tree replicated on every rank; each rollout batch is sharded over the
    ranks' sim ranges and all-reduced, so all ranks see identical counts and
    make identical choices, and the result equals dvc_mcts_search on one GPU
    (§R9, §P).  Returns (best_code, [(code, visits, wins)])."""
    return dvc.mcts_search_cb(state, sharded_batch(state, group), expansions, sims_per_child, seed, c=c,
                              max_depth=max_depth, flat=flat, crn=crn, informed=informed)
