"""Multi-GPU sharding of binding spaces (one process per GPU, torch.distributed).

SURVEY.md §8(e): bindings are partitioned across ranks — rank g evaluates its
contiguous pieces of the canonical (Appendix C) index space with the recorded
test sets replicated — so the data path needs no collective.  The only exchange
is the result, and it is ONE collective per sweep: every rank packs, per space,
(passing count, first passing index, reason histogram, a fixed-size prefix of its
passing indices) into one int64 tensor and a single all_gather_into_tensor hands
every rank every rank's block; the MIN of the first passing index (the candidate
the reference's rank-order loop, pipeline.cpp:248-310, would reach first), the
SUM of the histograms and the merge of the passing lists the host confirms with
P1 are then local.  With the "nccl" backend that is one NVLink collective; the
same code runs on "gloo" for the CPU tests.
"""
from __future__ import annotations

from typing import Callable

import numpy as np

NONE = (1 << 62)  # "no passing binding" sentinel
PREFIX = 32       # passing indices per (rank, space) carried by the packed block
_HDR = 2 + 5      # passing count, first passing index, reason histogram


def block_range(count: int, rank: int, world: int) -> tuple:
    """Contiguous block partition of [0, count)."""
    return count * rank // world, count * (rank + 1) // world


def pack(results: list, prefix: int = PREFIX) -> np.ndarray:
    """[(passing indices ascending, passing count, reason histogram)] per space ->
    int64 [n_spaces, 7 + prefix] (first = NONE when the rank found none)."""
    out = np.full((len(results), _HDR + prefix), -1, dtype=np.int64)
    for i, (passing, n, hist) in enumerate(results):
        p = np.asarray(passing, dtype=np.int64)
        out[i, 0] = int(n)
        out[i, 1] = int(p[0]) if n > 0 and len(p) else NONE
        out[i, 2:_HDR] = np.asarray(hist, dtype=np.int64)
        k = min(len(p), prefix)
        out[i, _HDR:_HDR + k] = p[:k]
    return out


def combine(blocks: np.ndarray, prefix: int = PREFIX) -> list:
    """int64 [world, n_spaces, 7 + prefix] -> [(sorted passing list, first passing
    index or -1, summed histogram, complete)] per space; complete is False when
    some rank had more passing indices than the prefix carries."""
    out = []
    for i in range(blocks.shape[1]):
        b = blocks[:, i, :]
        counts = b[:, 0]
        passing = sorted(int(x) for r in range(b.shape[0]) for x in b[r, _HDR:_HDR + min(int(counts[r]), prefix)])
        first = int(b[:, 1].min())
        out.append((passing, -1 if first == NONE else first, b[:, 2:_HDR].sum(axis=0),
                    bool((counts <= prefix).all())))
    return out


def reduce_packed(results: list, dist, device="cpu", prefix: int = PREFIX) -> list:
    """The per-sweep result exchange: one all_gather_into_tensor of the packed
    per-space blocks (see module doc).  Returns combine()'s list."""
    local = pack(results, prefix)
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return combine(local[None], prefix)
    import torch

    world = dist.get_world_size()
    src = torch.from_numpy(local).to(device)
    dst = torch.empty((world * src.shape[0], src.shape[1]), dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(dst, src)  # rank blocks concatenated along dim 0
    return combine(dst.cpu().numpy().reshape(world, src.shape[0], src.shape[1]), prefix)


def reduce_results(local_passing: list, local_hist: np.ndarray, dist, device="cpu") -> tuple:
    """One space: (sorted passing list, first passing index or -1, summed histogram)."""
    passing, first, hist, complete = reduce_packed([(list(local_passing), len(local_passing), local_hist)], dist,
                                                   device, prefix=max(PREFIX, _max_len(local_passing, dist)))[0]
    assert complete
    return passing, first, hist


def _max_len(local_passing, dist) -> int:
    """The longest passing list over ranks (a scalar MAX, so the packed prefix
    can carry every list of a one-space reduction)."""
    n = len(local_passing)
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return n
    import torch

    t = torch.tensor([n], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return int(t.item())


def sweep(count: int, evaluate: Callable[[int, int], tuple], dist=None, device="cpu") -> tuple:
    """evaluate(lo, hi) -> (passing indices, reason histogram) on this rank's block."""
    rank = dist.get_rank() if dist is not None and dist.is_initialized() else 0
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    lo, hi = block_range(count, rank, world)
    passing, hist = evaluate(lo, hi)
    return reduce_results(list(passing), hist, dist, device)


def sharded_step(jobs: list, shards: list, run_local: Callable[[], list], dist=None, device="cpu") -> list:
    """One multi-GPU sweep step as bench.py times it: this rank's pieces
    (`shards[i]` = [begin, end) of jobs[i], workloads.plan_shards) are evaluated by
    run_local() -> [(passing, count, hist)] per job (empty ranges contribute
    nothing), then the single packed all-gather.  Returns combine()'s list."""
    local = run_local()
    assert len(local) == len(jobs) == len(shards)
    return reduce_packed(local, dist, device)
