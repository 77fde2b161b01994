"""Sequence-sharded data parallelism for the LF-MMI loss.

Utterances are independent (batch independence is bitwise,
/root/reference/pkg/tests/test_forward_backward.py:168-180) and the objective
is additive over utterances (/root/reference/pkg/tests/test_loss.py:82-96),
so a batch splits across ranks with no data-path collective: every rank runs
``lfmmi_chain_loss`` on its own shard and the only exchange is one all-reduce
(sum) of the three f64 totals ``{sum_ok(num - den), sum_ok T_b, #failed}``
(``loss.py:61-72`` semantics are then applied to the global sums, so the
normalised loss equals the single-process one).  Gradients are never
exchanged: each rank's gradient is w.r.t. its own shard of network outputs.

One process per GPU; the process group is NCCL on B200 (NVLink 5 / NVSwitch)
and gloo in the CPU tests.
"""

from __future__ import annotations

import heapq

import numpy as np

__all__ = ["lpt_shards", "shard_of", "reduce_totals", "loss_from_totals"]


def lpt_shards(costs, world_size: int) -> list[np.ndarray]:
    """Longest-processing-time assignment of items to ``world_size`` ranks.

    ``costs[b]`` is the estimated work of item b (``T_b * (I_den + I_num,b)``,
    or simply ``T_b``).  Items are taken in decreasing cost (stable on ties),
    each to the currently least-loaded rank (lowest rank on ties), so every
    rank derives the same assignment without communication.  Each shard is
    returned in ascending item order (keeps the sorted-batch convention).
    """
    costs = np.asarray(costs, dtype=np.float64)
    if world_size < 1:
        raise ValueError(f"world_size must be >= 1, got {world_size}")
    order = np.argsort(-costs, kind="stable")
    heap = [(0.0, r) for r in range(world_size)]
    shards: list[list[int]] = [[] for _ in range(world_size)]
    for b in order:
        load, r = heapq.heappop(heap)
        shards[r].append(int(b))
        heapq.heappush(heap, (load + float(costs[b]), r))
    return [np.array(sorted(s), dtype=np.int64) for s in shards]


def shard_of(costs, rank: int, world_size: int) -> np.ndarray:
    """Item indices owned by ``rank`` under :func:`lpt_shards`."""
    if not 0 <= rank < world_size:
        raise ValueError(f"rank {rank} outside [0, {world_size})")
    return lpt_shards(costs, world_size)[rank]


def reduce_totals(totals, group=None):
    """All-reduce (sum) the 3-element f64 totals tensor in place and return it.

    With no initialised process group (single process) this is the identity.
    """
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(totals, op=dist.ReduceOp.SUM, group=group)
    return totals


def loss_from_totals(totals, batch_size: int, normalize_by_frames: bool = True):
    """(objective, loss, num_failed) from globally reduced totals (loss.py:61-72)."""
    tot = np.asarray(totals, dtype=np.float64).reshape(3)
    num_failed = int(round(tot[2]))
    if num_failed == batch_size:
        raise RuntimeError(f"all {batch_size} utterances failed numerically")
    objective = float(tot[0])
    frames = float(tot[1])
    loss = -objective / frames if normalize_by_frames else -objective
    return objective, loss, num_failed
