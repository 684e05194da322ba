"""GPU parity of the batched binding evaluator (libatc_b200 K0/K1/K2) against the
reference's own per-binding verify_rewrite verdicts (tests/golden, dumped from the
compiled reference) and against the CPU oracle.  Bit-exact: every binding's first
failing test and failure reason must be identical."""
import numpy as np
import pytest

from paper_2301_11659_b200 import Evaluator, fixtures
from paper_2301_11659_b200 import _lib as L

from . import oracle_lib as O

pytestmark = pytest.mark.gpu

STEMS = [s for s in fixtures.stems() if "specs" in fixtures.load(s).meta]


@pytest.fixture(scope="module")
def ev():
    return Evaluator()


def _check_explicit(ev, stem, sname, T=16, variant="testsets", which="p2"):
    p = fixtures.load(stem)
    v = p.verdicts(sname, which)
    space = p.space(sname)
    am, sm = space.decode(v["idx"])
    ts = p.testsets(T, variant=variant)
    got = ev.eval_bindings(fixtures.spec(sname), ts, am, sm)
    np.testing.assert_array_equal(got.fail_t, v["fail_t"], err_msg=f"{stem} x {sname}: first failing test")
    np.testing.assert_array_equal(got.reason, v["reason"], err_msg=f"{stem} x {sname}: reason")
    return got


@pytest.mark.parametrize("stem", STEMS)
def test_explicit_lists_match_reference(ev, stem):
    """Every binding the reference evaluated (full spaces up to 400k, samples of the
    2.3e9 conv spaces) gets the reference's exact (first failing t, reason) at T=16."""
    for sname in fixtures.load(stem).spec_names():
        _check_explicit(ev, stem, sname)


@pytest.mark.parametrize("stem", STEMS)
def test_parity_T10(ev, stem):
    """At T = verify_tests = 10 (pipeline.hpp:97) the verdict is the T=16 verdict
    truncated: pass iff the first failure is at t >= 10."""
    p = fixtures.load(stem)
    for sname in p.spec_names():
        v = p.verdicts(sname)
        space = p.space(sname)
        am, sm = space.decode(v["idx"])
        got = ev.eval_bindings(fixtures.spec(sname), p.testsets(10), am, sm)
        expect_pass = (v["fail_t"] < 0) | (v["fail_t"] >= 10)
        np.testing.assert_array_equal(got.reason == 0, expect_pass)


@pytest.mark.parametrize("stem", ["naive_f32", "naive_rowmajor"])
def test_config1_64cubed(ev, stem):
    """BASELINE configs[0]: P2 at m=n=k=64 with 16 sets (identity accepted for the
    row spec, the transposed binding for the col spec)."""
    for sname in ("gemm_rowmajor", "gemm_colmajor", "gemm_rowmajor_ld"):
        got = _check_explicit(ev, stem, sname, variant="testsets64", which="p2_64")
        # with m = n = k = 64 every size map of the right array permutation passes:
        # the identity perm block [0, 27) for the row spec, the A<->B swap block
        # [54, 81) (which holds the transposed binding 73) for the col spec
        if sname == "gemm_rowmajor":
            assert got.first_pass == 0 and got.ok[21] and got.ok[:27].all()
        if sname == "gemm_colmajor":
            assert got.first_pass == 54 and got.ok[73] and got.ok[54:81].all()


@pytest.mark.parametrize("stem,sname", [("naive_ld", "gemm_rowmajor_ld"), ("strassen_staged", "gemm_rowmajor"),
                                        ("gemm_square", "gemm_rowmajor"), ("naive_colmajor", "gemm_colmajor")])
def test_enumerated_matches_explicit(ev, stem, sname):
    """atc_eval_enumerated (device-side Appendix C decode) returns exactly the
    passing set and reason histogram of the reference dump."""
    p = fixtures.load(stem)
    v = p.verdicts(sname)
    assert v["enumerated"] == "full"
    space = p.space(sname)
    passing, n, hist = ev.eval_enumerated(fixtures.spec(sname), p.testsets(16), space)
    want = v["idx"][v["reason"] == 0]
    np.testing.assert_array_equal(passing, want)
    assert n == len(want)
    assert hist.tolist() == [int((v["reason"] == r).sum()) for r in range(5)]


def test_unpruned_accepted_sets_appendix_a(ev):
    """P2-accepted indices of the unpruned spaces (T=10)."""
    expect = {("naive_rowmajor", "gemm_rowmajor"): [21], ("naive_rowmajor", "gemm_colmajor"): [73],
              ("naive_colmajor", "gemm_rowmajor"): [73], ("strassen_staged", "gemm_rowmajor"): [21, 48],
              ("gemm_square", "gemm_rowmajor"): [0], ("naive_ld", "gemm_rowmajor_ld"): [44790],
              ("blocked_copy_local", "gemm_colmajor"): [181]}
    for (stem, sname), want in expect.items():
        p = fixtures.load(stem)
        passing, n, _ = ev.eval_enumerated(fixtures.spec(sname), p.testsets(10), p.space(sname))
        assert passing.tolist() == want, (stem, sname, passing)


@pytest.mark.parametrize("stem", ["naive_ld", "conv_direct", "kernel_axpy", "im2col_buffered"])
def test_gpu_matches_oracle_port(ev, stem):
    """Independent of the golden dump: the literal CPU restatement and the GPU agree."""
    p = fixtures.load(stem)
    rng = np.random.default_rng(1)
    for sname in p.spec_names():
        space = p.space(sname)
        idx = rng.choice(space.count, min(space.count, 3000), replace=False).astype(np.uint64)
        am, sm = space.decode(idx)
        ts = p.testsets(16)
        got = ev.eval_bindings(fixtures.spec(sname), ts, am, sm)
        ft, rs = O.verify_many(fixtures.spec(sname), ts, am, sm)
        np.testing.assert_array_equal(got.fail_t, ft)
        np.testing.assert_array_equal(got.reason, rs)


def test_empty_and_single(ev):
    p = fixtures.load("naive_rowmajor")
    spec = fixtures.spec("gemm_rowmajor")
    ts = p.testsets(4)
    got = ev.eval_bindings(spec, ts, np.zeros((0, 3), np.uint8), np.zeros((0, 3), np.uint8))
    assert len(got.reason) == 0 and got.first_pass == -1
    am, sm = p.space("gemm_rowmajor").decode([21])
    got = ev.eval_bindings(spec, ts, am, sm)
    assert got.reason.tolist() == [0] and got.first_pass == 0


def test_testset_failure_is_reason3(ev):
    """A test whose original run failed rejects every binding at that t (rewriter.cpp:247-251)."""
    p = fixtures.load("naive_rowmajor")
    ts = p.testsets(6)
    ts.test_ok[3] = 0
    ts._handles.clear()
    am, sm = p.space("gemm_rowmajor").decode([21])
    got = ev.eval_bindings(fixtures.spec("gemm_rowmajor"), ts, am, sm)
    assert got.fail_t.tolist() == [3] and got.reason.tolist() == [L.FAIL_TESTSET]


def test_malformed_spec_rejected(ev):
    p = fixtures.load("naive_rowmajor")
    spec = fixtures.spec("gemm_rowmajor")
    d = spec.to_desc()
    d.array_livein[0] = 0  # two outputs
    import ctypes as C

    h = p.testsets(2).upload(ev.ctx)
    am = np.zeros((1, 3), np.uint8)
    rc = L.lib().atc_eval_bindings(ev.ctx.handle, C.byref(d), h.value, am.ctypes.data, am.ctypes.data, 1, 0,
                                   am.ctypes.data, am.ctypes.data, None)
    assert rc == L.ATC_ERR_ARG
    assert b"output" in L.lib().atc_last_error(ev.ctx.handle)


@pytest.mark.parametrize("stem", STEMS)
def test_fp32_screen_mode_identical_verdicts(ev, stem):
    """ATC_MODE_FP32_SCREEN (FP32 FMA with the stated error bound, FP64 only for
    undecided positions) gives exactly the reference's verdicts."""
    p = fixtures.load(stem)
    for sname in p.spec_names():
        v = p.verdicts(sname)
        am, sm = p.space(sname).decode(v["idx"])
        got = ev.eval_bindings(fixtures.spec(sname), p.testsets(16), am, sm, mode=L.MODE_FP32_SCREEN)
        np.testing.assert_array_equal(got.fail_t, v["fail_t"])
        np.testing.assert_array_equal(got.reason, v["reason"])


@pytest.mark.parametrize("stem", ["naive_f32", "naive_rowmajor"])
def test_fp32_screen_mode_64cubed(ev, stem):
    for sname in ("gemm_rowmajor", "gemm_colmajor"):
        p = fixtures.load(stem)
        v = p.verdicts(sname, "p2_64")
        am, sm = p.space(sname).decode(v["idx"])
        got = ev.eval_bindings(fixtures.spec(sname), p.testsets(16, variant="testsets64"), am, sm,
                               mode=L.MODE_FP32_SCREEN)
        np.testing.assert_array_equal(got.fail_t, v["fail_t"])
        np.testing.assert_array_equal(got.reason, v["reason"])


def _shrunk(ts, lens):
    """The same tests with region p cut to lens[p] elements (None: unchanged)."""
    from paper_2301_11659_b200.evaluator import RecordedTestsets

    cut = lambda a, L: a if (a is None or L is None) else a[:L].copy()
    init = [[cut(a, lens[p]) for p, a in enumerate(row)] for row in ts.init]
    final = [None if row is None else [cut(a, lens[p]) for p, a in enumerate(row)] for row in ts.final]
    return RecordedTestsets(ts.params, ts.ints.copy(), init, final, ts.test_ok.copy(), seeds=ts.seeds, skips=ts.skips)


CONV_VARIANTS = {
    "recorded": lambda ts: ts,
    # small regions: dispatch failures (extent > region) and access-bound (UB) failures
    "in_3000": lambda ts: _shrunk(ts, [3000, None, None, None]),
    "in_700_out_900": lambda ts: _shrunk(ts, [700, None, 900, None]),
    "wt_200": lambda ts: _shrunk(ts, [None, 200, None, None]),
    # digit values < 1 (dispatch "size #q is not positive")
    "zero_int": lambda ts: _with_int(ts, 1, 0),
    "neg_int": lambda ts: _with_int(ts, 0, -3),
    "test0_failed": lambda ts: _with_ok(ts, 0),
    # a size above 200: 64-bit index arithmetic (the generic row screen)
    "big_int": lambda ts: _with_int(ts, 2, 300),
}


def _with_int(ts, i, v):
    ts = _shrunk(ts, [None] * 4)
    ts.ints[0, i] = v
    return ts


def _with_ok(ts, t):
    ts = _shrunk(ts, [None] * 4)
    ts.test_ok[t] = 0
    return ts


@pytest.mark.parametrize("variant", sorted(CONV_VARIANTS))
@pytest.mark.parametrize("stem", ["conv_direct", "im2col_buffered", "conv_permuted_sig"])
def test_enumerated_conv_matches_explicit(ev, stem, variant):
    """The enumerated conv screen (k_screen_conv_planes: digit-0 verdicts by
    thresholds) returns exactly the passing set and reason histogram of the
    explicit per-binding path (k_screen/k_confirm, itself pinned to the reference
    dumps) on whole row-unaligned ranges, including test sets that make the
    dispatch, access-bound and test-set reasons occur."""
    p = fixtures.load(stem)
    space = p.space("conv2d")
    spec = fixtures.spec("conv2d")
    ts = CONV_VARIANTS[variant](p.testsets(16))
    rng = np.random.default_rng(11)
    ranges = [(0, 1 << 19), (int(rng.integers(1, space.count - (1 << 20))), 654_321),
              (space.count - 100_003, space.count), (381367040, 381367049)]
    for b, e in ranges:
        e = b + e if e < b else e
        passing, n, hist = ev.eval_enumerated(spec, ts, space, b, e)
        idx = np.arange(b, e, dtype=np.uint64)
        am, sm = space.decode(idx)
        got = ev.eval_bindings(spec, ts, am, sm)
        want = idx[got.reason == 0]
        np.testing.assert_array_equal(passing, want, err_msg=f"{stem}/{variant} [{b},{e})")
        assert n == len(want)
        assert hist.tolist() == np.bincount(got.reason, minlength=5).tolist(), (stem, variant, b, e)
        print(stem, variant, b, e, hist.tolist())


GEMM_VARIANTS = {
    "recorded": lambda ts: ts,
    "int1_is_1": lambda ts: _with_int(ts, 1, 1),
    "int0_is_2": lambda ts: _with_int(ts, 0, 2),
    "int2_is_0": lambda ts: _with_int(ts, 2, 0),
    "c_300": lambda ts: _shrunk(ts, [None, None, 300, None]),
    "big_int": lambda ts: _with_int(ts, 1, 250),
}


@pytest.mark.parametrize("variant", sorted(GEMM_VARIANTS))
@pytest.mark.parametrize("stem", ["naive_ld", "kernel_dot", "blocked_copy_local", "naive_colmajor", "strassen_staged"])
def test_enumerated_gemm_matches_explicit(ev, stem, variant):
    """The enumerated gemm screen (k_screen_rows with the k_gemm_need written-set
    lookup) agrees with the explicit per-binding path on whole spaces, with test
    sets whose t = 0 sizes make partial, overlapping (ldc < n) and empty writes."""
    p = fixtures.load(stem)
    for sname in p.spec_names():
        space = p.space(sname)
        spec = fixtures.spec(sname)
        ts = GEMM_VARIANTS[variant](p.testsets(16))
        passing, n, hist = ev.eval_enumerated(spec, ts, space, 0, space.count)
        idx = np.arange(space.count, dtype=np.uint64)
        got = ev.eval_bindings(spec, ts, *space.decode(idx))
        want = idx[got.reason == 0]
        np.testing.assert_array_equal(passing, want, err_msg=f"{stem}/{sname}/{variant}")
        assert n == len(want)
        assert hist.tolist() == np.bincount(got.reason, minlength=5).tolist(), (stem, sname, variant)


def test_enumerated_many_matches_single(ev):
    """atc_eval_enumerated_many (all corpus spaces in one stream pass) returns per
    job exactly what atc_eval_enumerated returns for that job alone, including
    partial ranges, an empty range and a job with more passing bindings than cap."""
    from paper_2301_11659_b200 import workloads

    jobs = workloads.corpus_jobs()
    items = [(j.spec, j.ts, j.space, 0, j.count) for j in jobs]
    j0 = next(j for j in jobs if j.stem == "conv_direct")
    items += [(j0.spec, j0.ts, j0.space, 381367040, 381367049), (j0.spec, j0.ts, j0.space, 5, 5)]
    g = next(j for j in jobs if j.stem == "naive_rowmajor" and j.spec_name == "gemm_rowmajor")
    ts64 = fixtures.load("naive_rowmajor").testsets(16, variant="testsets64")
    items.append((g.spec, ts64, g.space, 0, g.count))  # 27 passing bindings, cap 8 below
    single = [ev.eval_enumerated(spec, ts, space, b, e, cap=8) for spec, ts, space, b, e in items]
    sweep = ev.sweep(items, cap=8)
    runs = [ev.eval_enumerated_many(items, cap=8)] + [sweep.run() for _ in range(3)]  # eager, then graph replays
    for many in runs:
        for (ps, ns, hs), (pm, nm, hm) in zip(single, many):
            np.testing.assert_array_equal(pm, ps)
            assert nm == ns and hm.tolist() == hs.tolist()
    sweep.close()


SCREEN_CASES = [("conv_direct", "in_700_out_900", 0, 1 << 21), ("conv_permuted_sig", "wt_200", 1234567, 1234567 + 999_999),
                ("im2col_buffered", "recorded", 0, None), ("conv_direct", "zero_int", 17, 2_000_017),
                ("winograd_1d", "in_3000", 5_000_000, 9_000_000)]


def test_conv_screen_kernels_agree():
    """k_screen_conv_pairs (default), k_screen_conv_planes (ATC_CONV_SCREEN_PLANES) and
    the generic k_screen_rows (ATC_CONV_SCREEN_GENERIC), selected per context with
    atc_set_option, give identical passing sets and reason histograms."""
    res = {}
    for name, opt in (("pairs", L.CONV_SCREEN_AUTO), ("planes", L.CONV_SCREEN_PLANES),
                      ("generic", L.CONV_SCREEN_GENERIC)):
        ctx = L.Context(0)
        ctx.set_option(L.OPT_CONV_SCREEN, opt)
        e = Evaluator(ctx)
        out = []
        for stem, variant, b, end in SCREEN_CASES:
            p = fixtures.load(stem)
            space = p.space("conv2d")
            ts = CONV_VARIANTS[variant](p.testsets(16))
            passing, n, hist = e.eval_enumerated(fixtures.spec("conv2d"), ts, space, b,
                                                 space.count if end is None else end)
            out.append((passing.tolist(), n, hist.tolist()))
        res[name] = out
        ctx.close()
    assert res["pairs"] == res["planes"] == res["generic"]
    assert any(r[2][4] for r in res["pairs"]) and any(r[2][2] for r in res["pairs"])


def test_set_option_rejects_bad_values(ev):
    with pytest.raises(L.AtcError):
        ev.ctx.set_option(L.OPT_CONV_SCREEN, 7)
    with pytest.raises(L.AtcError):
        ev.ctx.set_option(99, 0)


@pytest.mark.parametrize("stem", ["naive_f32", "conv_direct", "naive_ld", "im2col_buffered", "strassen_staged"])
def test_seeded_upload_regenerates_regions(ev, stem):
    """atc_testsets_upload_seeded rebuilds every probe image on the GPU from the
    tests' mt19937_64 streams (std::mt19937_64, uniform_real(-1,1), f32 rounding)
    bit-identically to the host regions, and the final images from the
    final-minus-init entries."""
    import ctypes as C

    p = fixtures.load(stem)
    ts = p.testsets(16)
    h = ts.upload_seeded(ev.ctx)
    nP, T, lens = len(ts.ptrs), ts.n_tests, [len(ts.init[0][q]) for q in range(len(ts.ptrs))]
    tot = T * sum(lens)
    ini, fin = np.empty(tot), np.empty(tot)
    L.check(ev.ctx.handle, L.lib().atc_testsets_download(ev.ctx.handle, C.c_void_p(h.value), ini.ctypes.data,
                                                         fin.ctypes.data))
    o = 0
    for t in range(T):
        for q in range(nP):
            if ts.test_ok[t]:
                assert np.array_equal(ini[o:o + lens[q]].view(np.uint64), np.asarray(ts.init[t][q]).view(np.uint64))
                assert np.array_equal(fin[o:o + lens[q]].view(np.uint64), np.asarray(ts.final[t][q]).view(np.uint64))
            o += lens[q]
    # the same verdicts through the seeded handle
    for sname in p.spec_names():
        space = p.space(sname)
        end = min(space.count, 1 << 22)
        want = ev.eval_enumerated(fixtures.spec(sname), ts, space, 0, end)
        ts2 = p.testsets(16)
        ts2._handles[id(ev.ctx)] = h
        got = ev.eval_enumerated(fixtures.spec(sname), ts2, space, 0, end)
        np.testing.assert_array_equal(got[0], want[0])
        assert got[1] == want[1] and got[2].tolist() == want[2].tolist()
    ts2._handles.clear()


def test_seeded_update_in_place_with_prepared_sweep(ev):
    """atc_testsets_update_seeded rewrites a handle's test sets in place; a
    prepared (graph-replayed) sweep over it then evaluates the new contents —
    re-captured when the new int values change the plan — exactly like a fresh
    one-shot evaluation of the same test sets."""
    import ctypes as C

    from paper_2301_11659_b200.evaluator import _TestsetHandle

    p = fixtures.load("conv_direct")
    base = p.testsets(16)
    h = base.upload_seeded(ev.ctx)
    space, spec = p.space("conv2d"), fixtures.spec("conv2d")
    ranges = [(0, 1 << 22), (381367000, 381367100)]
    holder = p.testsets(16)
    holder._handles[id(ev.ctx)] = h  # the sweep reads this handle
    sweep = ev.sweep([(spec, holder, space, b, e) for b, e in ranges])
    variants = [base, _with_int(base, 2, 5), _with_int(base, 4, 3), base]
    for ts in variants:
        s, keep = ts.seeded_struct()
        L.check(ev.ctx.handle, L.lib().atc_testsets_update_seeded(ev.ctx.handle, C.c_void_p(h.value), C.byref(s)))
        for _ in range(2):  # eager/capture, then replay
            got = sweep.run()
            for (b, e), (pg, ng, hg) in zip(ranges, got):
                pw, nw, hw = ev.eval_enumerated(spec, ts, space, b, e)
                np.testing.assert_array_equal(pg, pw)
                assert ng == nw and hg.tolist() == hw.tolist()
    sweep.close()
    holder._handles.clear()


@pytest.mark.parametrize("stem", ["conv_direct", "im2col_virtual", "naive_ld", "strassen_staged", "naive_f32"])
def test_seeded_needed_only_regions(ev, stem):
    """needed_only seeded handles (only the region prefixes an evaluation can read
    are generated) give the same verdicts as whole regions: full spaces (or their
    first 2^22 bindings) and an explicit list with every reason code; downloading
    such a handle is refused."""
    import ctypes as C

    p = fixtures.load(stem)
    ts = p.testsets(16)
    h = ts.upload_seeded(ev.ctx, needed_only=True)
    holder = p.testsets(16)
    holder._handles[id(ev.ctx)] = h
    for sname in p.spec_names():
        space, spec = p.space(sname), fixtures.spec(sname)
        end = min(space.count, 1 << 22)
        want = ev.eval_enumerated(spec, ts, space, 0, end)
        got = ev.eval_enumerated(spec, holder, space, 0, end)
        np.testing.assert_array_equal(got[0], want[0])
        assert got[1] == want[1] and got[2].tolist() == want[2].tolist()
        idx = np.arange(0, end, max(1, end // 4096), dtype=np.uint64)
        am, sm = space.decode(idx)
        a, b = ev.eval_bindings(spec, ts, am, sm), ev.eval_bindings(spec, holder, am, sm)
        np.testing.assert_array_equal(a.fail_t, b.fail_t)
        np.testing.assert_array_equal(a.reason, b.reason)
    buf = np.empty(ts.n_tests * sum(len(ts.init[0][q]) for q in range(len(ts.ptrs))))
    with pytest.raises(L.AtcError, match="prefixes"):
        L.check(ev.ctx.handle, L.lib().atc_testsets_download(ev.ctx.handle, C.c_void_p(h.value), buf.ctypes.data,
                                                             None))
    holder._handles.clear()


@pytest.mark.parametrize("stem", ["conv_direct", "im2col_buffered", "naive_ld", "strassen_staged", "naive_f32",
                                  "conv_stride2"])
def test_prefix_upload_regions(ev, stem):
    """atc_testsets_upload_prefix (the host's own probe images, only the needed
    prefixes cross PCIe) gives the same verdicts as the full-region upload: full
    spaces (or their first 2^22 bindings) and a strided explicit list."""
    p = fixtures.load(stem)
    ts = p.testsets(16)
    h = ts.upload_prefix(ev.ctx)
    holder = p.testsets(16)
    holder._handles[id(ev.ctx)] = h
    for sname in p.spec_names():
        space, spec = p.space(sname), fixtures.spec(sname)
        end = min(space.count, 1 << 22)
        want = ev.eval_enumerated(spec, ts, space, 0, end)
        got = ev.eval_enumerated(spec, holder, space, 0, end)
        np.testing.assert_array_equal(got[0], want[0])
        assert got[1] == want[1] and got[2].tolist() == want[2].tolist()
        idx = np.arange(0, end, max(1, end // 4096), dtype=np.uint64)
        am, sm = space.decode(idx)
        a, b = ev.eval_bindings(spec, ts, am, sm), ev.eval_bindings(spec, holder, am, sm)
        np.testing.assert_array_equal(a.fail_t, b.fail_t)
        np.testing.assert_array_equal(a.reason, b.reason)
    holder._handles.clear()
    h.free()


def test_eval_bindings_many_equals_single(ev):
    """atc_eval_bindings_many over several (spec, test-set handle, list) jobs of
    different sizes equals atc_eval_bindings on each job alone (verdicts and
    first passing index); an empty job and a job with a malformed list are
    reported per job."""
    import ctypes as C

    jobs, keep = [], []
    for stem, sname, stride in (("naive_ld", "gemm_rowmajor_ld", 37), ("naive_rowmajor", "gemm_colmajor", 1),
                                ("conv_direct", "conv2d", 1 << 20), ("naive_f32", "gemm_rowmajor", 1)):
        p = fixtures.load(stem)
        ts, space, spec = p.testsets(16), p.space(sname), fixtures.spec(sname)
        idx = np.arange(0, space.count, stride, dtype=np.uint64)[:5000]
        am, sm = space.decode(idx)
        jobs.append((spec, ts, np.ascontiguousarray(am), np.ascontiguousarray(sm)))
    arr = (L.BindJob * (len(jobs) + 1))()
    for i, (spec, ts, am, sm) in enumerate(jobs):
        n = am.shape[0]
        ft, rs, desc = np.empty(n, np.int8), np.empty(n, np.int8), spec.to_desc()
        keep.append((ft, rs, desc))
        j = arr[i]
        j.spec = C.cast(C.pointer(desc), C.c_void_p)
        j.ts = ts.upload(ev.ctx).value
        j.arr_map, j.size_map, j.n_bindings = am.ctypes.data, sm.ctypes.data, n
        j.fail_t, j.reason = ft.ctypes.data, rs.ctypes.data
    e = arr[len(jobs)]  # empty job
    e.spec, e.ts, e.n_bindings = arr[0].spec, arr[0].ts, 0
    L.check(ev.ctx.handle, L.lib().atc_eval_bindings_many(ev.ctx.handle, arr, len(jobs) + 1, 0))
    for i, (spec, ts, am, sm) in enumerate(jobs):
        want = ev.eval_bindings(spec, ts, am, sm)
        np.testing.assert_array_equal(keep[i][0], want.fail_t)
        np.testing.assert_array_equal(keep[i][1], want.reason)
        assert arr[i].first_pass == want.first_pass and arr[i].status == 0
    assert arr[len(jobs)].status == 0 and arr[len(jobs)].first_pass == -1
    bad = (L.BindJob * 1)()
    bad[0].spec, bad[0].ts, bad[0].n_bindings = arr[0].spec, arr[0].ts, 4  # no maps
    assert L.lib().atc_eval_bindings_many(ev.ctx.handle, bad, 1, 0) == L.ATC_ERR_ARG and bad[0].status == L.ATC_ERR_ARG


def test_seeded_update_many_batched(ev):
    """atc_testsets_update_seeded_many over several distinct needed_only handles (the
    batched path: one staging copy, k_copy_meta + k_probe_regions_many for all of them)
    rewrites every handle exactly as a fresh evaluation of the new test sets sees it."""
    import ctypes as C

    stems = ["conv_direct", "naive_ld", "im2col_virtual", "naive_f32"]
    progs = [fixtures.load(s) for s in stems]
    bases = [p.testsets(16) for p in progs]
    handles, holders = [], []
    for p, base in zip(progs, bases):  # first contents: another int value at t = 2
        h = _with_int(base, 2, 5).upload_seeded(ev.ctx, needed_only=True)
        holder = p.testsets(16)
        holder._handles[id(ev.ctx)] = h
        handles.append(h)
        holders.append(holder)
    for rnd in range(2):  # twice: the second reuses the staging buffers
        structs, keeps = zip(*[b.seeded_struct(needed_only=True) for b in bases])
        arr = (L.SeededTestsets * len(structs))(*structs)
        hp = (C.c_void_p * len(handles))(*[h.value for h in handles])
        L.check(ev.ctx.handle, L.lib().atc_testsets_update_seeded_many(ev.ctx.handle, hp, arr, len(handles)))
        for stem, p, base, holder in zip(stems, progs, bases, holders):
            for sname in p.spec_names():
                space, spec = p.space(sname), fixtures.spec(sname)
                end = min(space.count, 1 << 22)
                want = ev.eval_enumerated(spec, base, space, 0, end)
                got = ev.eval_enumerated(spec, holder, space, 0, end)
                np.testing.assert_array_equal(got[0], want[0])
                assert got[1] == want[1] and got[2].tolist() == want[2].tolist(), (stem, sname, rnd)
    for holder in holders:
        holder._handles.clear()
