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
    except BaseException as e:  # report instead of leaving the parent waiting
        q.put((rank, repr(e), None, None, None, None, None))
        raise
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
        assert pr.exitcode == 0, res
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


BENCH_STEMS = ("naive_rowmajor", "naive_colmajor", "blocked_mult4", "vec8_unguarded", "naive_f32")


def _bench_flow_worker(rank, world, port, q):
    """bench.py's multi-GPU step on CPU: workloads.plan_shards pieces, a stub
    evaluator (the CPU oracle on this rank's pieces), shard.sharded_step's single
    packed all-gather."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2301_11659_b200 import shard, workloads
        from tests import oracle_lib as O

        jobs = [j for j in workloads.corpus_jobs(16, ("gemm",)) if j.stem in BENCH_STEMS]
        workloads.BIG_SPACE = 600  # force the cost-model split of the larger spaces
        shards = workloads.plan_shards(jobs, rank, world)

        def run_local():
            out = []
            for j, (b, e) in zip(jobs, shards):
                idx = np.arange(b, e, dtype=np.uint64)
                if len(idx) == 0:
                    out.append((np.zeros(0, np.uint64), 0, np.zeros(5, np.int64)))
                    continue
                _, rs = O.verify_many(j.spec, j.ts, *j.space.decode(idx), threads=2)
                p = idx[rs == 0]
                out.append((p, len(p), np.bincount(rs.astype(np.int64), minlength=5)))
            return out

        combined = shard.sharded_step(jobs, shards, run_local, dist)
        q.put((rank, [(pl, first, hist.tolist(), ok) for pl, first, hist, ok in combined], shards,
               [(j.count, j.expected_pass) for j in jobs]))
    except BaseException as e:  # report instead of leaving the parent waiting
        q.put((rank, repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_two_rank_bench_flow():
    """Both ranks end the step with the same combined result, equal to the
    reference's single-process passing sets (T=16) for every space, every binding
    evaluated exactly once, and some space really split across the two ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_flow_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0, res
    (_, comb0, sh0, meta), (_, comb1, sh1, _) = res
    assert comb0 == comb1
    split = 0
    for (pl, first, hist, ok), (count, exp), a, b in zip(comb0, meta, sh0, sh1):
        assert ok and pl == exp and first == (exp[0] if exp else -1)
        assert sum(hist) == count and hist[0] == len(exp)
        assert (a[1] - a[0]) + (b[1] - b[0]) == count
        split += (a[1] > a[0]) and (b[1] > b[0])
    assert split >= 1


def test_packed_reduce_roundtrip():
    """shard.pack / combine: MIN of first, SUM of histograms, merged passing
    lists, and the overflow flag when a rank's list exceeds the prefix."""
    from paper_2301_11659_b200 import shard

    r0 = [([5, 9], 2, [1, 2, 3, 0, 0]), ([], 0, [0, 4, 0, 0, 0])]
    r1 = [([3], 1, [1, 0, 0, 1, 0]), (list(range(40)), 40, [40, 0, 0, 0, 0])]
    blocks = np.stack([shard.pack(r0), shard.pack(r1)])
    (p0, f0, h0, c0), (p1, f1, h1, c1) = shard.combine(blocks)
    assert p0 == [3, 5, 9] and f0 == 3 and h0.tolist() == [2, 2, 3, 1, 0] and c0
    assert f1 == 0 and not c1 and h1.tolist() == [40, 4, 0, 0, 0]


def test_c_plan_equals_python_plan():
    """atc_plan_shards (the library's shard plan, used by atc_group_*) is the same
    rule as workloads.plan_shards for every rank of N = 1, 2, 3, 4, 8 on the corpus
    spaces and on synthetic mixes (host arithmetic: runs without a GPU)."""
    from types import SimpleNamespace

    from paper_2301_11659_b200 import group, workloads

    corpus = [j.count for j in workloads.corpus_jobs()]
    rng = np.random.default_rng(7)
    mixes = [corpus, [1 << 30, 1 << 24, 5, (1 << 24) - 1, 9 * (1 << 30), 3],
             [int(x) for x in rng.integers(1, 1 << 34, size=23)] + [int(x) for x in rng.integers(1, 1 << 20, size=9)]]
    for counts in mixes:
        jobs = [SimpleNamespace(count=c) for c in counts]
        for world in (1, 2, 3, 4, 8):
            cplan = group.plan_shards(counts, world)
            for r in range(world):
                assert cplan[r] == [tuple(x) for x in workloads.plan_shards(jobs, r, world)], (world, r)
