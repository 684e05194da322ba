"""Benchmark workloads (BASELINE.json configs) built from the recorded corpus.

corpus  every GEMM and conv2d corpus program x every spec of its class, the FULL
        unpruned binding space with 16 recorded P2 test
        sets each (configs 2-4; the conv spaces are 2.3e9-9.3e9 bindings, which
        only a GPU can sweep).
stress  naive_ld x gemm_rowmajor_ld, 279,936 bindings x 16 sets (config 4 alone).
naive64 naive_f32 x {gemm_rowmajor, gemm_colmajor} at m = n = k = 64 (config 1:
        the P2 sets drawn with the [64, 64] rule, 162 bindings per spec).
pruned  the ranked (pruned) candidate list of every program (config 2 as the
        pipeline sees it; latency-bound): pruned_lists().

Algorithmic bytes: a screened (binding, t) pair is charged
elem_bytes * (ext_A + ext_B + ext_C) with ext_X = prod of X's API dims under
the binding's decoded sizes.  Over an enumerated space this sum factorises:
sum over size maps of prod_{q in dims(X)} u[s_q] = (sum_i u_i)^|dims X| * nI^(nS-|dims X|).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import fixtures
from .evaluator import BindingSpace, RecordedTestsets
from .spec import ApiSpec


@dataclass
class Job:
    stem: str
    spec_name: str
    spec: ApiSpec
    space: BindingSpace
    ts: RecordedTestsets
    expected_pass: list | None  # reference P2-passing indices (T=16) when the dump is full

    @property
    def count(self) -> int:
        return self.space.count

    def t0_bytes(self, begin: int, end: int) -> float:
        """Algorithmic bytes of screening [begin, end) at t = 0 (closed form,
        proportional within a permutation block)."""
        sp, sz = self.spec, self.space
        u = self.ts.ints[0].astype(np.float64)
        nI, nS = len(u), len(sp.size_params())
        size_idx = {p.name: q for q, p in enumerate(sp.size_params())}
        is_f32 = [p.elem == "f32" for p in self.ts.ptrs]
        total = 0.0
        per_perm = []
        for perm in sz.perms:
            b = 0.0
            for a, arr in enumerate(sp.arrays()):
                dims = [size_idx[d] for d in arr.dims]
                # distinct size params per array in the bundled specs
                assert len(set(dims)) == len(dims)
                ext_sum = u.sum() ** len(dims) * float(nI) ** (nS - len(dims))
                b += (4.0 if is_f32[perm[a]] else 8.0) * ext_sum
            per_perm.append(b / sz.size_maps)
        per_perm = np.array(per_perm)
        # bytes per binding is constant within a permutation block
        pm = sz.size_maps
        for p, bpb in enumerate(per_perm):
            lo, hi = max(begin, p * pm), min(end, (p + 1) * pm)
            if hi > lo:
                total += bpb * (hi - lo)
        return total

    def t0_flops(self, begin: int, end: int) -> float:
        """2 * MACs of computing the full t=0 output (upper bound on screened work)."""
        sp = self.spec
        u = self.ts.ints[0].astype(np.float64)
        nI, nS = len(u), len(sp.size_params())
        roles = {p.role for p in sp.size_params()}
        if sp.semantics == "gemm":
            k = 3  # m, n, k
        else:
            k = 7 if {"oh", "ow"} <= roles else 5
        return 2.0 * (u.sum() ** k * float(nI) ** (nS - k) / self.space.size_maps) * (end - begin)


def corpus_jobs(T: int = 16, kinds=("gemm", "conv")) -> list:
    jobs = []
    for stem in fixtures.stems():
        p = fixtures.load(stem)
        if "specs" not in p.meta or p.meta.get("corpus_dir") not in kinds:
            continue
        ts = p.testsets(T)
        for sname in p.spec_names():
            v = p.verdicts(sname)
            exp = None
            if v["enumerated"] == "full":
                ok = (v["fail_t"] < 0) | (v["fail_t"] >= T)
                exp = v["idx"][ok].tolist()
            jobs.append(Job(stem, sname, fixtures.spec(sname), p.space(sname), ts, exp))
    return jobs


@dataclass
class SpaceCount:
    """A corpus binding space described without its test sets (pure arithmetic:
    no probe image is regenerated, so nothing touches libatc_b200)."""

    stem: str
    spec_name: str
    spec: ApiSpec
    count: int


def corpus_spaces(kinds=("gemm", "conv")) -> list:
    """corpus_jobs()' spaces (same order), counts only."""
    out = []
    for stem in fixtures.stems():
        p = fixtures.load(stem)
        if "specs" not in p.meta or p.meta.get("corpus_dir") not in kinds:
            continue
        for sname in p.spec_names():
            out.append(SpaceCount(stem, sname, fixtures.spec(sname), p.space(sname).count))
    return out


def naive64_jobs(T: int = 16) -> list:
    """Config 1: naive_f32 at 64^3 (the testsets64 variant: P2 sets drawn with
    m = n = k = [64, 64]) against both dense GEMM specs, full 162-binding spaces."""
    p = fixtures.load("naive_f32")
    ts = p.testsets(T, variant="testsets64")
    jobs = []
    for sname in ("gemm_rowmajor", "gemm_colmajor"):
        v = p.verdicts(sname, "p2_64")
        ok = (v["fail_t"] < 0) | (v["fail_t"] >= T)
        jobs.append(Job("naive_f32", sname, fixtures.spec(sname), p.space(sname), ts, v["idx"][ok].tolist()))
    return jobs


def pruned_lists(T: int = 16) -> list:
    """Config 2 as the pipeline sees it: per (program, spec) the ranked candidate
    list find_matchings + rank_candidates produced (tests/golden, from the
    reference), as (stem, spec, testsets, arr_map, size_map, reference P2 ok)."""
    from .evaluator import encode_bindings

    out = []
    for stem in fixtures.stems():
        p = fixtures.load(stem)
        if "specs" not in p.meta or p.meta.get("corpus_dir") not in ("gemm", "conv"):
            continue
        ts = None
        for sname, s in p.meta["specs"].items():
            ranked = s.get("pruned") or []
            if not ranked or s.get("truncated"):
                continue
            ts = ts or p.testsets(T)
            spec = fixtures.spec(sname)
            am, sm = encode_bindings(ranked, spec, p.user_ptrs, p.user_ints)
            space = p.space(sname)
            v = p.verdicts(sname)
            pos = {int(g): i for i, g in enumerate(v["idx"])}
            ok = []
            for c in ranked:
                g = pos.get(space.index_of(c))
                ok.append(None if g is None else bool(v["fail_t"][g] < 0 or v["fail_t"][g] >= T))
            out.append((stem, sname, spec, ts, am, sm, ok))
    return out


def stress_jobs(T: int = 16) -> list:
    return [j for j in corpus_jobs(T, ("gemm",)) if j.stem == "naive_ld" and j.spec_name == "gemm_rowmajor_ld"]


def shard(count: int, rank: int, world: int) -> tuple:
    """Contiguous block partition of [0, count)."""
    return count * rank // world, count * (rank + 1) // world


BIG_SPACE = 1 << 24  # spaces at least this large are split by the cost model below

# Per-space cost model of a large (conv) space on one B200, from the measured chain
# (tools/rank_breakdown.py, r2 kernels): a fixed part (position tables, K2, finalize:
# ~0.10 ms) plus the K1 screen (~0.123 ms per 2.32e9 bindings).  csrc/group.cu carries
# the same constants (atc_plan_shards).
SPACE_FIXED_MS = 0.10
SPACE_MS_PER_BINDING = 0.123 / 2324522934


def space_cost_ms(n: int) -> float:
    return SPACE_FIXED_MS + n * SPACE_MS_PER_BINDING if n > 0 else 0.0


def plan_shards(jobs: list, rank: int, world: int) -> list:
    """This rank's [begin, end) of every job.

    Large spaces are balanced with the cost model, largest first: the target per
    rank is their total cost / world; a space goes whole to the least-loaded rank
    if that stays within the target (+15%), else it is cut into the fewest k ~equal
    contiguous pieces (k <= world, one per least-loaded rank) that do, else into the
    k with the lowest resulting maximum — a rank pays the fixed part of every piece
    it takes, so a space is split only when that buys balance.  Small spaces — chains of a few latency-bound kernels — go whole to one
    rank each, dealt round-robin.  Ranks without a piece of a space get an empty
    range (and contribute nothing to its reduction).  Deterministic: every rank
    computes the same plan."""
    if world == 1:
        return [(0, j.count) for j in jobs]
    big = [i for i, j in enumerate(jobs) if j.count >= BIG_SPACE]
    target = sum(space_cost_ms(jobs[i].count) for i in big) / world
    load = [0.0] * world
    pieces = {}
    for i in sorted(big, key=lambda i: (-jobs[i].count, i)):
        n = jobs[i].count
        order = sorted(range(world), key=lambda r: (load[r], r))
        # the fewest pieces that keep every receiving rank within the target (+15%),
        # else the piece count with the lowest resulting maximum
        fits, best = None, None
        for k in range(1, world + 1):
            peak = load[order[k - 1]] + space_cost_ms(-(-n // k))
            if fits is None and peak <= 1.15 * target:
                fits = k
            if best is None or peak < best[0] - 1e-12:
                best = (peak, k)
        k = fits or best[1]
        ranks = sorted(order[:k])
        pieces[i] = {}
        for idx, r in enumerate(ranks):
            b, e = shard(n, idx, k)
            pieces[i][r] = (b, e)
            load[r] += space_cost_ms(e - b)
    out, k = [], 0
    for i, j in enumerate(jobs):
        if i in pieces:
            out.append(pieces[i].get(rank, (0, 0)))
        else:
            out.append((0, j.count) if k % world == rank else (0, 0))
            k += 1
    return out
