"""Extended semantics: gemm_ext (transA/transB, alpha/beta,
lda/ldb/ldc) and conv2d_ext (stride, zero padding, dilation) — no reference
counterpart, so parity is pinned by known answers computed independently
(oracle/gen_ext_kats.py: numpy products on transposed views, padded / strided /
dilated windows; exact binary fractions) and then GPU == CPU statement
(oracle/ext_oracle.c) bit for bit on the recorded corpus test sets."""
import json
import os

import numpy as np
import pytest

from paper_2301_11659_b200 import ext, fixtures

from . import oracle_lib as O

KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ext_known_answers.json")))["cases"]


def _bufs(case):
    return [np.asarray([np.nan if x is None else x for x in b], dtype=np.float64) for b in case["bufs"]]


def _same(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray([np.nan if x is None else x for x in b], dtype=np.float64)
    return np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("case", KATS, ids=[c["name"] for c in KATS])
def test_oracle_known_answers(case):
    bufs = _bufs(case)
    rc, detail = O.run_ext(ext.spec(case["spec"]), case["sizes"], case["floats"], bufs, case["is_f32"])
    assert rc == case["status"], detail
    if rc:
        assert case.get("why", "") in detail
    for got, want in zip(bufs, case["expect"]):
        assert _same(got, want), (case["name"], got, want)


def test_spaces_and_encoding():
    """The extended space of a gemm program: the base Appendix C digits plus the
    trans / alpha / beta digits; decode and binding agree."""
    p = fixtures.load("naive_ld")
    sp = ext.space_of(p, ext.spec("gemm_ext"))
    nI = len(p.user_ints)
    assert sp.count == 6 * nI ** 6 * 2 * 2 * 2 * 2  # perms x sizes x trans x (alpha, beta: constants)
    idx = np.array([0, 1, 2, sp.count - 1, 12345], dtype=np.uint64)
    am, sm, fm = sp.decode(idx)
    b = sp.binding(12345)
    assert set(b["sizes"]) == {q.name for q in sp.spec.size_params()}
    assert b["sizes"]["tc_transa"] in (0, 1) and b["floats"]["tc_alpha"] in (1.0, 0.0)
    assert (sm[:, 0] >= nI).all() and (sm[:, 2] < nI).all()


@pytest.mark.gpu
@pytest.mark.parametrize("case", KATS, ids=[c["name"] for c in KATS])
def test_gpu_known_answers(case):
    from paper_2301_11659_b200 import AtcError, default_context

    bufs = _bufs(case)
    if case["status"]:
        with pytest.raises(AtcError):
            ext.run_reference_ext(default_context(), ext.spec(case["spec"]), case["sizes"], case["floats"], bufs,
                                  case["is_f32"])
    else:
        ext.run_reference_ext(default_context(), ext.spec(case["spec"]), case["sizes"], case["floats"], bufs,
                              case["is_f32"])
    for got, want in zip(bufs, case["expect"]):
        assert _same(got, want), (case["name"], got, want)


def _sample(sp, n, seed, extra=()):
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([rng.integers(0, sp.count, n, dtype=np.uint64),
                                    np.asarray(extra, dtype=np.uint64)]))
    return idx


EXT_CASES = [("naive_ld", "gemm_ext", 20000), ("naive_colmajor", "gemm_ext", 20000), ("naive_f32", "gemm_ext", 8000),
             ("kernel_axpy", "gemm_ext", 8000), ("conv_direct", "conv2d_ext", 6000),
             ("conv_stride2", "conv2d_ext", 6000), ("winograd_1d", "conv2d_ext", 3000)]


@pytest.mark.gpu
@pytest.mark.parametrize("stem,sname,n", EXT_CASES)
def test_gpu_matches_oracle_on_corpus_test_sets(stem, sname, n):
    """GPU vs the CPU statement: identical first failing test and reason for every
    sampled binding of the extended space, on the program's recorded test sets."""
    from paper_2301_11659_b200 import default_context

    p = fixtures.load(stem)
    sp = ext.space_of(p, ext.spec(sname))
    ts = p.testsets(16)
    idx = _sample(sp, n, 7)
    am, sm, fm = sp.decode(idx)
    ft, rs, _ = ext.eval_bindings_ext(default_context(), sp.spec, ts, am, sm, fm)
    oft, ors = O.verify_ext_many(sp.spec, ts, am, sm, fm)
    np.testing.assert_array_equal(rs, ors)
    np.testing.assert_array_equal(ft, oft)
    assert len(set(rs.tolist())) >= 2


@pytest.mark.gpu
def test_conv_stride2_lifts_with_stride_binding():
    """conv_stride2 computes a stride-2 convolution (h = 2*oh + r - 2), which the
    reference's conv2d cannot express (P1 and P2 reject it).
    Under conv2d_ext the reference's own pruned binding plus stride (2, 2), pad 0,
    dil 1 passes all 16 recorded tests (GPU and CPU statement agree), and the same
    binding with stride 1 fails."""
    from paper_2301_11659_b200 import default_context

    p = fixtures.load("conv_stride2")
    sp = ext.space_of(p, ext.spec("conv2d_ext"))
    base = p.space("conv2d")
    b0 = base.binding(int(p.meta["specs"]["conv2d"]["pruned_index"][0]))
    ts = p.testsets(16)
    rows = []
    for stride in (2, 1):
        am, sm, fm = _encode(sp, b0, {"tc_stride_h": stride, "tc_stride_w": stride, "tc_pad_h": 0, "tc_pad_w": 0,
                                      "tc_dil_h": 1, "tc_dil_w": 1})
        rows.append((am, sm, fm))
    am, sm, fm = (np.concatenate([r[i] for r in rows]) for i in range(3))
    ft, rs, first = ext.eval_bindings_ext(default_context(), sp.spec, ts, am, sm, fm)
    oft, ors = O.verify_ext_many(sp.spec, ts, am, sm, fm)
    assert rs.tolist() == ors.tolist() and ft.tolist() == oft.tolist()
    assert rs[0] == 0 and first == 0 and rs[1] != 0


def _encode(sp, base_binding: dict, consts: dict):
    """ABI maps of one extended binding: the base binding's arrays and user-int
    sizes plus the given constants."""
    nI = len(sp.user_ints)
    am = np.array([[sp.user_ptrs.index(base_binding["arrays"][a.name]) for a in sp.spec.arrays()]], dtype=np.uint8)
    sm = np.zeros((1, sp.nS), dtype=np.uint8)
    for q, prm in enumerate(sp.spec.size_params()):
        if prm.name in consts:
            sm[0, q] = nI + sp.iconst.index(consts[prm.name])
        else:
            sm[0, q] = sp.user_ints.index(base_binding["sizes"][prm.name])
    fm = np.zeros((1, sp.nF), dtype=np.uint8)
    return am, sm, fm
