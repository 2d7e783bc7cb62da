"""Multi-GPU mining: one process per GPU, pairs sharded, ordered gather.

Document pairs are independent (align.py:402-448), so the only
cross-device step is the final ordered gather of mined rows: each rank
mines a contiguous range of the input pairs -- balanced by N*M cells --
on its own GPU, and rank 0 concatenates the per-rank results in rank
order, which is input order.  There is no collective on the data path;
`torch.distributed` (NCCL between GPUs, gloo in the CPU tests) carries
only the gather of the small result lists.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from .align import MiningConfig, MiningOutcome, _shard_bounds


def shard_range(weights: np.ndarray, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of pairs owned by `rank` (cell-balanced)."""
    bounds = _shard_bounds(np.asarray(weights, dtype=np.int64), world)
    while len(bounds) < world:  # fewer pairs than ranks: trailing ranks get nothing
        bounds.append((bounds[-1][1], bounds[-1][1]))
    return bounds[rank]


def pair_weights(pairs: Sequence) -> np.ndarray:
    return np.array([len(p.source.sentences) * len(p.target.sentences) for p in pairs], dtype=np.int64)


def mine_corpus_distributed(model, lexicon, pairs: Sequence, config: MiningConfig, engine: str = "nw_wavefront",
                            group=None, dst: int = 0,
                            mine_fn: Callable | None = None) -> MiningOutcome | None:
    """mine_corpus over all ranks of `group`; returns the full outcome on
    rank `dst` (None elsewhere).  Every rank passes the same `pairs`.

    `mine_fn(model, lexicon, pairs, config, engine)` mines a rank's shard
    (default: align.mine_corpus on the rank's current CUDA device)."""
    import torch.distributed as dist

    from .align import mine_corpus

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    lo, hi = shard_range(pair_weights(pairs), rank, world)
    fn = mine_fn or mine_corpus
    local = fn(model, lexicon, list(pairs[lo:hi]), config, engine)
    payload = (rank, local.rows, local.failures)
    gathered = [None] * world if rank == dst else None
    dist.gather_object(payload, gathered, dst=dst, group=group)
    if rank != dst:
        return None
    gathered.sort(key=lambda x: x[0])
    rows = tuple(r for _, rs, _ in gathered for r in rs)
    failures = tuple(f for _, _, fs in gathered for f in fs)
    return MiningOutcome(rows=rows, failures=failures)
