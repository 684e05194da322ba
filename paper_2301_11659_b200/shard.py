"""Multi-GPU sharding of binding spaces (one process per GPU, torch.distributed).

SURVEY.md §8(e): bindings are block-partitioned across ranks — rank g evaluates
[g*B/G, (g+1)*B/G) of the canonical (Appendix C) index space with the recorded
test sets replicated — so the data path needs no collective.  The only exchange
is the result: one all-reduce MIN of the first passing index (the candidate the
reference's rank-order loop, pipeline.cpp:248-310, would reach first) and an
all-gather of the (tiny) passing lists the host confirms with P1.  With the
"nccl" backend these are NVLink collectives; the same code runs on "gloo" for
the CPU tests.
"""
from __future__ import annotations

from typing import Callable

import numpy as np

NONE = (1 << 62)  # "no passing binding" sentinel for the MIN reduction


def block_range(count: int, rank: int, world: int) -> tuple:
    """Contiguous block partition of [0, count)."""
    return count * rank // world, count * (rank + 1) // world


def reduce_results(local_passing: list, local_hist: np.ndarray, dist, device="cpu") -> tuple:
    """Combine per-rank (passing indices, reason histogram) into the global
    (sorted passing list, first passing index or -1, summed histogram)."""
    import torch

    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        first = min(local_passing) if local_passing else -1
        return sorted(local_passing), first, np.asarray(local_hist)
    first = torch.tensor([min(local_passing) if local_passing else NONE], dtype=torch.int64, device=device)
    dist.all_reduce(first, op=dist.ReduceOp.MIN)
    hist = torch.tensor(np.asarray(local_hist, dtype=np.int64), device=device)
    dist.all_reduce(hist, op=dist.ReduceOp.SUM)
    gathered = [None] * dist.get_world_size()
    dist.all_gather_object(gathered, list(map(int, local_passing)))
    passing = sorted(x for g in gathered for x in g)
    f = int(first.item())
    return passing, (-1 if f == NONE else f), hist.cpu().numpy()


def sweep(count: int, evaluate: Callable[[int, int], tuple], dist=None, device="cpu") -> tuple:
    """evaluate(lo, hi) -> (passing indices, reason histogram) on this rank's block."""
    rank = dist.get_rank() if dist is not None and dist.is_initialized() else 0
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    lo, hi = block_range(count, rank, world)
    passing, hist = evaluate(lo, hi)
    return reduce_results(list(passing), hist, dist, device)
