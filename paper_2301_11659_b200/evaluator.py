"""Batched candidate-binding evaluation on the GPU (host-side mirror).

Mirrors the reference's P2 surface rewriter::verify_rewrite
(/root/reference/proj/include/liftc/rewriter.hpp:77-80, src/rewriter.cpp:215-284)
for a whole batch of candidate bindings, and the pipeline's candidate loop rule
(src/pipeline.cpp:248-310): the winner is the first binding, in rank order, that
the host's P1 (equivalence::check_equivalence) calls Equivalent and that passes
P2.  P2 for every candidate runs here, on the GPU, through libatc_b200's C ABI;
P1 stays with the host that owns the interpreter.

Binding spaces follow SURVEY.md Appendix C (the canonical enumeration of the
unpruned space whose size matching::raw_candidate_count, matching.cpp:211-225,
reports).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from .probe import PROBE_REGION_LEN, SizeRules, p2_test_inputs
from .spec import ApiSpec


# ------------------------------------------------------------------ test sets --
@dataclass
class RecordedTestsets:
    """The binding-independent half of verify_rewrite for one function.

    ints[t, i]       user int param i at test t (signature order)
    init[t][p]       probe-image region of user pointer p (float64, f32-rounded for *f32)
    final[t][p]      the same region after the original run
    test_ok[t]       False if draw_sizes failed or the original run was not Normal
    """

    params: list  # [Param] in signature order
    ints: np.ndarray  # int64 [T, nI]
    init: list  # [T][nP] float64 arrays
    final: list  # [T][nP] float64 arrays (None when not test_ok)
    test_ok: np.ndarray  # int32 [T]
    _handles: dict = field(default_factory=dict, repr=False)
    # how verify_rewrite drew the initial regions (when known): test t's Rng seed and
    # the stream position of each region's first draw — atc_testsets_upload_seeded
    seeds: Optional[np.ndarray] = None  # uint64 [T]
    skips: Optional[np.ndarray] = None  # uint64 [T, nP]
    # the user float params (signature order) as build_probe_image drew them — read
    # only by the extended semantics (paper_2301_11659_b200/ext.py)
    floats: Optional[np.ndarray] = None  # float64 [T, nF]

    @property
    def ptrs(self) -> list:
        return [p for p in self.params if p.kind == "ptr"]

    @property
    def int_params(self) -> list:
        return [p.name for p in self.params if p.kind == "int"]

    @property
    def n_tests(self) -> int:
        return int(self.ints.shape[0])

    def head(self, T: int) -> "RecordedTestsets":
        """The first T tests (t-indexed streams are independent: prefix = fewer tests)."""
        return RecordedTestsets(self.params, self.ints[:T].copy(), self.init[:T], self.final[:T],
                                self.test_ok[:T].copy(),
                                seeds=None if self.seeds is None else self.seeds[:T].copy(),
                                skips=None if self.skips is None else self.skips[:T].copy())

    def seeded_struct(self, needed_only: bool = False, _streams: bool = True):
        """atc_seeded_testsets: seeds + stream positions + the final-minus-init
        entries (positions where the original run's final image differs).
        needed_only: the device generates only the region prefixes an evaluation
        can read (include/atc_b200.h)."""
        if _streams and (self.seeds is None or self.skips is None):
            raise ValueError("these test sets carry no stream seeds")
        ptrs = self.ptrs
        T, nP = self.n_tests, len(ptrs)
        pos, val, off = [], [], [0]
        for t in range(T):
            for p in range(nP):
                if self.final[t] is not None:
                    d = np.nonzero(self.final[t][p] != self.init[t][p])[0]
                    pos.append(d.astype(np.int32))
                    val.append(np.asarray(self.final[t][p])[d].astype(np.float64))
                    off.append(off[-1] + len(d))
                else:
                    off.append(off[-1])
        dpos = np.ascontiguousarray(np.concatenate(pos) if pos else np.zeros(0, np.int32), dtype=np.int32)
        dval = np.ascontiguousarray(np.concatenate(val) if val else np.zeros(0), dtype=np.float64)
        doff = np.array(off, dtype=np.int64)
        ints = np.ascontiguousarray(self.ints, dtype=np.int64)
        is_f32 = np.array([1 if p.elem == "f32" else 0 for p in ptrs], dtype=np.int32)
        lens = np.array([len(self.init[0][p]) for p in range(nP)], dtype=np.int64)
        ok = np.ascontiguousarray(self.test_ok, dtype=np.int32)
        seeds = np.ascontiguousarray(self.seeds if _streams else np.zeros(T), dtype=np.uint64)
        skips = np.ascontiguousarray(self.skips if _streams else np.zeros((T, nP)), dtype=np.uint64)
        s = _lib.SeededTestsets()
        s.n_tests, s.n_ints, s.n_ptrs = T, ints.shape[1], nP
        s.int_values = ints.ctypes.data
        s.ptr_is_f32 = is_f32.ctypes.data
        s.region_len = lens.ctypes.data
        s.test_ok = ok.ctypes.data
        s.stream_seed = seeds.ctypes.data
        s.stream_skip = skips.ctypes.data
        s.diff_off = doff.ctypes.data
        s.diff_pos = dpos.ctypes.data
        s.diff_val = dval.ctypes.data
        s.needed_only = 1 if needed_only else 0
        return s, [ints, is_f32, lens, ok, seeds, skips, doff, dpos, dval]

    def upload_seeded(self, ctx: "_lib.Context", needed_only: bool = False):
        """atc_testsets_upload_seeded: regions generated on the GPU from the seeds."""
        s, keep = self.seeded_struct(needed_only)
        out = C.c_void_p()
        _lib.check(ctx.handle, _lib.lib().atc_testsets_upload_seeded(ctx.handle, C.byref(s), C.byref(out)))
        h = _TestsetHandle(ctx, out.value)
        h.keep = keep  # host buffers stay valid until the handle is used (async upload)
        return h

    def upload_prefix(self, ctx: "_lib.Context"):
        """atc_testsets_upload_prefix: the host's own regions, of which only the
        prefixes an evaluation can read (+ the final-minus-init entries) cross PCIe."""
        s, keep = self.seeded_struct(needed_only=True, _streams=False)
        ints, is_f32, lens, ok, _, _, doff, dpos, dval = keep
        T, nP = self.n_tests, len(self.ptrs)
        init_ptrs = (C.c_void_p * (T * nP))()
        regions = []
        for t in range(T):
            for p in range(nP):
                if ok[t]:
                    a = np.ascontiguousarray(self.init[t][p], dtype=np.float64)
                    regions.append(a)
                    init_ptrs[t * nP + p] = a.ctypes.data
        px = _lib.PrefixTestsets()
        px.n_tests, px.n_ints, px.n_ptrs = s.n_tests, s.n_ints, s.n_ptrs
        px.int_values, px.ptr_is_f32, px.region_len, px.test_ok = s.int_values, s.ptr_is_f32, s.region_len, s.test_ok
        px.init = C.cast(init_ptrs, C.c_void_p)
        px.diff_off, px.diff_pos, px.diff_val = s.diff_off, s.diff_pos, s.diff_val
        out = C.c_void_p()
        _lib.check(ctx.handle, _lib.lib().atc_testsets_upload_prefix(ctx.handle, C.byref(px), C.byref(out)))
        return _TestsetHandle(ctx, out.value)

    def c_struct(self):
        ptrs = self.ptrs
        T, nP = self.n_tests, len(ptrs)
        keep = []
        ints = np.ascontiguousarray(self.ints, dtype=np.int64)
        is_f32 = np.array([1 if p.elem == "f32" else 0 for p in ptrs], dtype=np.int32)
        lens = np.array([len(self.init[0][p]) for p in range(nP)], dtype=np.int64)
        init_ptrs = (C.c_void_p * (T * nP))()
        fin_ptrs = (C.c_void_p * (T * nP))()
        for t in range(T):
            for p in range(nP):
                a = np.ascontiguousarray(self.init[t][p], dtype=np.float64)
                keep.append(a)
                init_ptrs[t * nP + p] = a.ctypes.data
                f = self.final[t][p] if self.final[t] is not None else None
                if f is not None:
                    f = np.ascontiguousarray(f, dtype=np.float64)
                    keep.append(f)
                    fin_ptrs[t * nP + p] = f.ctypes.data
                else:
                    fin_ptrs[t * nP + p] = None
        ok = np.ascontiguousarray(self.test_ok, dtype=np.int32)
        s = _lib.Testsets()
        s.n_tests, s.n_ints, s.n_ptrs = T, ints.shape[1], nP
        if self.floats is not None and self.floats.size:
            fl = np.ascontiguousarray(self.floats, dtype=np.float64)
            keep.append(fl)
            s.n_floats, s.float_values = fl.shape[1], fl.ctypes.data
        s.int_values = ints.ctypes.data_as(C.POINTER(C.c_int64))
        s.ptr_is_f32 = is_f32.ctypes.data_as(C.POINTER(C.c_int32))
        s.region_len = lens.ctypes.data_as(C.POINTER(C.c_int64))
        s.init = C.cast(init_ptrs, C.POINTER(C.c_void_p))
        s.final_ = C.cast(fin_ptrs, C.POINTER(C.c_void_p))
        s.test_ok = ok.ctypes.data_as(C.POINTER(C.c_int32))
        keep += [ints, is_f32, lens, init_ptrs, fin_ptrs, ok]
        return s, keep

    def upload(self, ctx: "_lib.Context"):
        """atc_testsets_upload: regions to HBM once, dirty lists built on the GPU."""
        h = self._handles.get(id(ctx))
        if h is not None:
            return h
        s, keep = self.c_struct()
        out = C.c_void_p()
        _lib.check(ctx.handle, _lib.lib().atc_testsets_upload(ctx.handle, C.byref(s), C.byref(out)))
        del keep
        h = _TestsetHandle(ctx, out.value)
        self._handles[id(ctx)] = h
        return h


class _TestsetHandle:
    def __init__(self, ctx, value):
        self.ctx, self.value = ctx, value

    def free(self):
        if self.value and self.ctx.handle:
            _lib.lib().atc_testsets_free(self.ctx.handle, self.value)
        self.value = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def record_testsets(function: str, params: list, rules: SizeRules, p2seed: int, tests: int,
                    run_original: Callable) -> RecordedTestsets:
    """Builds the T recorded test sets exactly as verify_rewrite draws them
    (rewriter.cpp:235-251).  `run_original(t, sizes, regions, floats)` is the
    host's interpreter run of the original function; it returns the final regions
    (dict name -> float64 array) or None when the run is not Normal."""
    ptrs = [p for p in params if p.kind == "ptr"]
    int_names = [p.name for p in params if p.kind == "int"]
    T = tests
    ints = np.zeros((T, len(int_names)), dtype=np.int64)
    float_names = [p.name for p in params if p.kind == "float"]
    floats = np.zeros((T, len(float_names)), dtype=np.float64)
    init, final, ok = [], [], np.zeros(T, dtype=np.int32)
    seeds, skips = np.zeros(T, dtype=np.uint64), np.zeros((T, len(ptrs)), dtype=np.uint64)
    for t in range(T):
        pt = p2_test_inputs(function, params, rules, p2seed, t)
        if pt.ok:
            floats[t] = [pt.floats[n] for n in float_names]
        if not pt.ok:
            init.append([np.zeros(PROBE_REGION_LEN) for _ in ptrs])
            final.append(None)
            continue
        ints[t] = [pt.sizes[n] for n in int_names]
        seeds[t] = pt.seed
        skips[t] = [pt.streams[p.name] for p in ptrs]
        init.append([pt.regions[p.name] for p in ptrs])
        fin = run_original(t, pt.sizes, pt.regions, pt.floats)
        if fin is None:
            final.append(None)
            continue
        final.append([fin[p.name] for p in ptrs])
        ok[t] = 1
    return RecordedTestsets(params, ints, init, final, ok, seeds=seeds, skips=skips, floats=floats)


# ------------------------------------------------------------- binding spaces --
class BindingSpace:
    """injective array maps (odometer order of
    matching.cpp:141-194 without filters) x functional size maps, global index =
    perm * |I|^|S| + s with size param q -> I[(s / |I|^q) % |I|]."""

    def __init__(self, user_ptrs: list, user_ints: list, spec: ApiSpec):
        self.user_ptrs, self.user_ints = list(user_ptrs), list(user_ints)
        self.api_arrays = [p.name for p in spec.arrays()]
        self.api_sizes = [p.name for p in spec.size_params()]
        perms = []
        nA, nU = len(self.api_arrays), len(self.user_ptrs)
        used, sel = [False] * nU, [0] * nA

        def rec(i):
            if i == nA:
                perms.append(list(sel))
                return
            for j in range(nU):
                if used[j]:
                    continue
                used[j] = True
                sel[i] = j
                rec(i + 1)
                used[j] = False

        if nA <= nU:
            rec(0)
        self.perms = np.array(perms, dtype=np.uint8).reshape(len(perms), nA)
        self.size_maps = len(self.user_ints) ** len(self.api_sizes)
        self.count = len(perms) * self.size_maps

    def decode(self, idx) -> tuple:
        idx = np.asarray(idx, dtype=np.uint64)
        perm = idx // np.uint64(self.size_maps)
        s = idx - perm * np.uint64(self.size_maps)
        arr = self.perms[perm.astype(np.int64)]
        nI = np.uint64(len(self.user_ints))
        sm = np.zeros((len(idx), len(self.api_sizes)), dtype=np.uint8)
        for q in range(len(self.api_sizes)):
            sm[:, q] = (s % nI).astype(np.uint8)
            s = s // nI
        return arr, sm

    def binding(self, idx: int) -> dict:
        arr, sm = self.decode([idx])
        return {"arrays": {a: self.user_ptrs[arr[0, i]] for i, a in enumerate(self.api_arrays)},
                "sizes": {a: self.user_ints[sm[0, q]] for q, a in enumerate(self.api_sizes)}, "scalars": {}}

    def index_of(self, binding: dict) -> int:
        sel = [self.user_ptrs.index(binding["arrays"][a]) for a in self.api_arrays]
        p = next(i for i, row in enumerate(self.perms.tolist()) if row == sel)
        s, mul = 0, 1
        for a in self.api_sizes:
            s += self.user_ints.index(binding["sizes"][a]) * mul
            mul *= len(self.user_ints)
        return p * self.size_maps + s


def encode_bindings(bindings: list, spec: ApiSpec, user_ptrs: list, user_ints: list) -> tuple:
    """CandidateBinding maps (api -> user name) into arr_map/size_map index rows."""
    arrays, sizes = spec.arrays(), spec.size_params()
    am = np.zeros((len(bindings), len(arrays)), dtype=np.uint8)
    sm = np.zeros((len(bindings), len(sizes)), dtype=np.uint8)
    for b, cb in enumerate(bindings):
        for a, p in enumerate(arrays):
            am[b, a] = user_ptrs.index(cb["arrays"][p.name])
        for q, p in enumerate(sizes):
            sm[b, q] = user_ints.index(cb["sizes"][p.name])
    return am, sm


# ---------------------------------------------------------------- evaluation --
@dataclass
class BatchVerdicts:
    fail_t: np.ndarray  # int8: first failing test, -1 when every test passed
    reason: np.ndarray  # int8: _lib.PASS / FAIL_*
    first_pass: int  # smallest passing index (rank), -1 if none

    @property
    def ok(self) -> np.ndarray:
        return self.reason == _lib.PASS


class Evaluator:
    """GPU P2 evaluator bound to one device context."""

    def __init__(self, ctx: Optional["_lib.Context"] = None, device: int = 0):
        self.ctx = ctx or _lib.default_context(device)

    def eval_bindings(self, spec: ApiSpec, ts: RecordedTestsets, arr_map: np.ndarray, size_map: np.ndarray,
                      mode: int = _lib.MODE_FP64, handle=None) -> BatchVerdicts:
        """`handle`: an already uploaded test-set handle of `ts` (e.g. upload_seeded)."""
        h = handle or ts.upload(self.ctx)
        n = int(arr_map.shape[0])
        am = np.ascontiguousarray(arr_map, dtype=np.uint8)
        sm = np.ascontiguousarray(size_map, dtype=np.uint8)
        ft = np.empty(n, dtype=np.int8)
        rs = np.empty(n, dtype=np.int8)
        first = C.c_int64(-1)
        desc = spec.to_desc()
        _lib.check(self.ctx.handle, _lib.lib().atc_eval_bindings(
            self.ctx.handle, C.byref(desc), h.value, am.ctypes.data, sm.ctypes.data, n, mode,
            ft.ctypes.data, rs.ctypes.data, C.byref(first)))
        return BatchVerdicts(ft, rs, int(first.value))

    def eval_enumerated(self, spec: ApiSpec, ts: RecordedTestsets, space: BindingSpace, begin: int = 0,
                        end: Optional[int] = None, cap: int = 1 << 16, mode: int = _lib.MODE_FP64):
        """Returns (passing indices (ascending), total passing, reason histogram)."""
        h = ts.upload(self.ctx)
        end = space.count if end is None else end
        surv = np.zeros(max(cap, 1), dtype=np.uint64)
        nsurv = C.c_int64(0)
        hist = np.zeros(5, dtype=np.int64)
        perms = np.ascontiguousarray(space.perms, dtype=np.uint8)
        desc = spec.to_desc()
        _lib.check(self.ctx.handle, _lib.lib().atc_eval_enumerated(
            self.ctx.handle, C.byref(desc), h.value, perms.ctypes.data, int(perms.shape[0]), begin, end, mode,
            surv.ctypes.data, cap, C.byref(nsurv), hist.ctypes.data))
        n = int(nsurv.value)
        return surv[:min(n, cap)].copy(), n, hist

    def eval_enumerated_many(self, items: list, cap: int = 1 << 16, mode: int = _lib.MODE_FP64) -> list:
        """eval_enumerated for many (spec, ts, space, begin, end) at once
        (atc_eval_enumerated_many: one stream pass, one result copy)."""
        return EnumSweep(self, items, cap, mode, prepared=False).run()

    def sweep(self, items: list, cap: int = 1 << 16, mode: int = _lib.MODE_FP64) -> "EnumSweep":
        """A prepared, reusable sweep (atc_enum_batch_*): run() repeatedly replays
        one CUDA graph of every job after the first eager run."""
        return EnumSweep(self, items, cap, mode, prepared=True)


class EnumSweep:
    def __init__(self, ev: Evaluator, items: list, cap: int, mode: int, prepared: bool):
        self.ev, self.cap, self.mode, self.n = ev, cap, mode, len(items)
        self.jobs = (_lib.EnumJob * max(self.n, 1))()
        self._keep = []
        for j, (spec, ts, space, begin, end) in enumerate(items):
            h = ts.upload(ev.ctx)
            desc = spec.to_desc()
            perms = np.ascontiguousarray(space.perms, dtype=np.uint8)
            surv = np.zeros(max(cap, 1), dtype=np.uint64)
            self._keep.append((desc, perms, surv, ts))
            jb = self.jobs[j]
            jb.spec = C.cast(C.pointer(desc), C.c_void_p)
            jb.ts = h.value
            jb.perms = perms.ctypes.data
            jb.n_perms = int(perms.shape[0])
            jb.begin, jb.end = int(begin), int(space.count if end is None else end)
            jb.survivors = surv.ctypes.data
            jb.cap = cap
        self._out = _lib.out_view(self.jobs, self.n, ["n_survivors", "reason_counts", "status"])
        self._surv = [k[2] for k in self._keep]
        self.handle = None
        if prepared:
            L = _lib.lib()
            self.handle = L.atc_enum_batch_create(ev.ctx.handle, self.jobs, self.n, mode)
            if not self.handle:
                raise _lib.AtcError(_lib.ATC_ERR_ARG, L.atc_last_error(ev.ctx.handle).decode())

    def run(self) -> list:
        """[(passing indices ascending (<= cap), passing count, reason histogram)] per item."""
        L = _lib.lib()
        if self.handle:
            _lib.check(self.ev.ctx.handle, L.atc_enum_batch_run(self.ev.ctx.handle, self.handle))
        else:
            _lib.check(self.ev.ctx.handle, L.atc_eval_enumerated_many(self.ev.ctx.handle, self.jobs, self.n,
                                                                      self.mode))
        # the jobs' out fields through one structured view of the ctypes array (per-job
        # ctypes attribute reads cost ~4 us each: 0.4 ms per 89-job step)
        st = self._out["status"]
        if st.any():
            j = int(np.flatnonzero(st)[0])
            raise _lib.AtcError(int(st[j]), f"job {j}: atc error {int(st[j])}")
        ks = self._out["n_survivors"].tolist()  # (slices past a buffer's cap end at the cap)
        return list(zip([s[:k].copy() for s, k in zip(self._surv, ks)], ks, list(self._out["reason_counts"].copy())))

    def close(self):
        if self.handle:
            _lib.lib().atc_enum_batch_destroy(self.ev.ctx.handle, self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class VerifyResult:
    """rewriter::VerifyResult (rewriter.hpp:69-73)."""

    ok: bool = False
    tests_run: int = 0
    detail: str = ""


def verify_rewrite_batch(function: str, bindings: list, spec: ApiSpec, ts: RecordedTestsets, user_ptrs: list,
                         evaluator: Optional[Evaluator] = None) -> list:
    """verify_rewrite for every binding at once; tests_run/detail follow
    rewriter.cpp:241-283 (tests_run = t + 1 after a mismatch, t after a
    dispatch failure)."""
    ev = evaluator or Evaluator()
    am, sm = encode_bindings(bindings, spec, user_ptrs, ts.int_params)
    v = ev.eval_bindings(spec, ts, am, sm)
    out = []
    out_array = next(p.name for p in spec.arrays() if p.liveness != "livein")
    for b, cb in enumerate(bindings):
        t, r = int(v.fail_t[b]), int(v.reason[b])
        if r == _lib.PASS:
            out.append(VerifyResult(True, ts.n_tests, ""))
        elif r == _lib.FAIL_MISMATCH:
            out.append(VerifyResult(False, t + 1, f"mismatch on {cb['arrays'][out_array]} at test {t}"))
        elif r == _lib.FAIL_DISPATCH:
            out.append(VerifyResult(False, t, f"dispatch failed: extent check at test {t}"))
        elif r == _lib.FAIL_TESTSET:
            out.append(VerifyResult(False, t, f"test {t}: could not draw sizes or original run failed"))
        else:
            out.append(VerifyResult(False, t, f"access outside a region at test {t}"))
    return out

