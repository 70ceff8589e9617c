"""paper_2403_10720_b200 -- B200-native batched Da Vinci Code MCTS rollouts
(arXiv 2403.10720, BASELINE.json north_star).

    from paper_2403_10720_b200 import dvc
    st = dvc.encode(obs_json)                 # SURVEY §8(a) a0, host
    codes = st.legal_actions()
    hist = dvc.rollout_batch_ex(st, codes, seed, 0, 0, n)   # a1-a5 on the GPU
    from paper_2403_10720_b200 import dist    # a6: sim-range sharding + NCCL all_reduce

The compute path is libdvc.so (include/dvc.h): hand-written sm_100a kernels.
"""

from . import dvc  # noqa: F401

__all__ = ["dvc"]
