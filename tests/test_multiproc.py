"""The N>1 path on CPU: world_size 2 over gloo (torch.distributed), each rank
evaluating its block of the naive_ld x gemm_rowmajor_ld space (279,936
bindings) with the CPU oracle; the combined result must equal the reference's
single-process verdicts (one passing binding, index 44790)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2301_11659_b200 import fixtures, shard
        from tests import oracle_lib as O

        p = fixtures.load("naive_ld")
        spec = fixtures.spec("gemm_rowmajor_ld")
        space = p.space("gemm_rowmajor_ld")
        ts = p.testsets(10)
        # keep the CPU cost small: every 7th binding plus the accepted one
        sub = np.unique(np.concatenate([np.arange(0, space.count, 7), [44790]])).astype(np.uint64)

        def evaluate(lo, hi):
            idx = sub[(sub >= lo) & (sub < hi)]
            am, sm = space.decode(idx)
            ft, rs = O.verify_many(spec, ts, am, sm, threads=2)
            hist = np.bincount(rs.astype(np.int64), minlength=5)
            return idx[rs == 0].tolist(), hist

        lo, hi = shard.block_range(space.count, rank, world)
        passing, first, hist = shard.sweep(space.count, evaluate, dist)
        q.put((rank, lo, hi, passing, first, hist.tolist(), len(sub)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sweep():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    (_, lo0, hi0, pass0, first0, hist0, n), (_, lo1, hi1, pass1, first1, hist1, _) = res
    assert lo0 == 0 and hi0 == lo1 and hi1 == 279936  # block partition covers the space once
    assert pass0 == pass1 == [44790] and first0 == first1 == 44790
    assert hist0 == hist1 and sum(hist0) == n and hist0[0] == 1


def test_block_range_partition():
    from paper_2301_11659_b200.shard import block_range

    for count in (0, 1, 7, 279936, 2324522934):
        for world in (1, 2, 3, 8):
            ranges = [block_range(count, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert max(h - l for l, h in ranges) - min(h - l for l, h in ranges) <= 1


def test_plan_shards_cover_every_space_once():
    """workloads.plan_shards: across ranks every binding of every corpus space is
    assigned exactly once in contiguous pieces; small spaces go whole to one rank
    and are dealt evenly; the large spaces' modelled cost is balanced (no rank above
    the per-rank target by more than one space's fixed part plus one piece)."""
    from paper_2301_11659_b200 import workloads

    jobs = workloads.corpus_jobs()
    for world in (1, 2, 4, 8):
        plans = [workloads.plan_shards(jobs, r, world) for r in range(world)]
        for i, j in enumerate(jobs):
            rs = sorted((plans[r][i] for r in range(world)), key=lambda x: x[0])
            covered = sum(e - b for b, e in rs)
            assert covered == j.count, (j.stem, world)
            nonempty = [(b, e) for b, e in rs if e > b]
            assert nonempty[0][0] == 0 and all(a[1] == c[0] for a, c in zip(nonempty, nonempty[1:]))
            if j.count < workloads.BIG_SPACE:
                assert len(nonempty) == 1
        big = [i for i, j in enumerate(jobs) if j.count >= workloads.BIG_SPACE]
        loads = [sum(workloads.space_cost_ms(plans[r][i][1] - plans[r][i][0]) for i in big) for r in range(world)]
        target = sum(workloads.space_cost_ms(jobs[i].count) for i in big) / world
        biggest = max(workloads.space_cost_ms(jobs[i].count) for i in big)
        assert max(loads) <= target + biggest, (world, loads)
        if world > 1:
            assert max(loads) < sum(loads) / 2 or world == 2
        small = [sum(1 for i, j in enumerate(jobs) if j.count < workloads.BIG_SPACE and plans[r][i][1] > 0)
                 for r in range(world)]
        assert max(small) - min(small) <= 1
