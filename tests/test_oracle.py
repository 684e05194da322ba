"""Pins the CPU oracle and the host-side input builder to the reference (CPU only).

Anchors:
  * equivalence_test.cpp:76-121 frozen run_reference vectors
  * seeds (Rng::mix, rng.hpp:32-44) and regenerated probe regions vs the golden dump
  * per-binding verify_rewrite verdicts dumped from the compiled reference
    (oracle/_ref/ref_tool golden) for every GEMM/conv corpus program
"""
import numpy as np
import pytest

from paper_2301_11659_b200 import fixtures
from paper_2301_11659_b200.probe import rng_mix

from . import oracle_lib as O


def _fnv_check(region, meta):
    assert O.fnv1a(region) == int(meta["init_fnv"])


# ---------------------------------------------------------------- frozen vectors
def test_frozen_rowmajor():  # equivalence_test.cpp:76-86
    c = np.zeros(4)
    assert O.run_reference(fixtures.spec("gemm_rowmajor"), [2, 2, 2], [np.array([1., 2, 3, 4]),
                                                                        np.array([5., 6, 7, 8]), c]) == 0
    assert c.tolist() == [19, 22, 43, 50]


def test_frozen_colmajor():  # :88-98
    c = np.zeros(4)
    O.run_reference(fixtures.spec("gemm_colmajor"), [2, 2, 2], [np.array([1., 3, 2, 4]), np.array([5., 7, 6, 8]), c])
    assert c.tolist() == [19, 43, 22, 50]


def test_frozen_strided_padding():  # :100-110
    c = np.array([0., 0, -9, 0, 0, -9])
    O.run_reference(fixtures.spec("gemm_rowmajor_ld"), [2, 2, 2, 3, 3, 3],
                    [np.array([1., 2, -9, 3, 4, -9]), np.array([5., 6, -9, 7, 8, -9]), c])
    assert c.tolist() == [19, 22, -9, 43, 50, -9]


def test_frozen_conv_ones():  # :112-121
    out = np.zeros(4)
    O.run_reference(fixtures.spec("conv2d"), [1, 1, 3, 3, 1, 2, 2, 2, 2], [np.ones(9), np.ones(4), out])
    assert out.tolist() == [4, 4, 4, 4]


# ---------------------------------------------------------------- seeds / inputs
@pytest.mark.parametrize("stem", fixtures.stems())
def test_seeds(stem):
    p = fixtures.load(stem)
    fseed = rng_mix(0, f"{p.meta['file']}:{p.function}")  # pipeline.cpp:131
    assert fseed == int(p.meta["fseed"])
    assert rng_mix(fseed, "post") == p.p2seed  # pipeline.cpp:277


@pytest.mark.parametrize("stem", ["naive_ld", "naive_f32", "conv_direct", "strassen_staged", "kernel_axpy",
                                  "blocked_mult4", "winograd_1d", "conv_stride2"])
def test_regenerated_probe_images(stem):
    """draw_sizes + build_probe_image restated (probe.py) reproduce the reference's
    sizes and every 65,536-element region bit-for-bit (FNV-1a of the raw bytes)."""
    p = fixtures.load(stem)
    ts = p.testsets(16, check=_fnv_check)
    assert ts.n_tests == 16


def test_regenerated_probe_images_64():
    p = fixtures.load("naive_f32")
    ts = p.testsets(16, variant="testsets64", check=_fnv_check)
    assert (ts.ints == 64).all()


# ---------------------------------------------------------------- binding spaces
@pytest.mark.parametrize("stem", fixtures.stems())
def test_binding_space_matches_reference(stem):
    """Appendix C enumeration: counts = matching::raw_candidate_count and the
    pruned candidates decode to the indices the reference dump computed."""
    p = fixtures.load(stem)
    for sname, s in (p.meta.get("specs") or {}).items():
        space = p.space(sname)
        assert space.count == s["count"] == s["raw"]
        for cand, idx in zip(s["pruned"], s["pruned_index"]):
            assert space.index_of(cand) == idx
            b = space.binding(idx)
            assert b["arrays"] == cand["arrays"] and b["sizes"] == cand["sizes"]


def _oracle_vs_golden(stem, sname, T=16, limit=None):
    p = fixtures.load(stem)
    v = p.verdicts(sname)
    idx = v["idx"]
    if limit is not None and len(idx) > limit:
        sel = np.random.default_rng(0).choice(len(idx), limit, replace=False)
        sel.sort()
    else:
        sel = np.arange(len(idx))
    space = p.space(sname)
    am, sm = space.decode(idx[sel])
    ts = p.testsets(T)
    ft, rs = O.verify_many(fixtures.spec(sname), ts, am, sm)
    np.testing.assert_array_equal(ft, v["fail_t"][sel])
    np.testing.assert_array_equal(rs, v["reason"][sel])
    return int((rs == 0).sum())


GEMM_STEMS = [s for s in fixtures.stems() if fixtures.load(s).meta.get("corpus_dir") == "gemm"
              and "specs" in fixtures.load(s).meta]
CONV_STEMS = [s for s in fixtures.stems() if fixtures.load(s).meta.get("corpus_dir") == "conv"
              and "specs" in fixtures.load(s).meta]


@pytest.mark.parametrize("stem", GEMM_STEMS)
def test_oracle_matches_reference_p2_gemm(stem):
    """The literal verify_rewrite restatement agrees with the reference on every
    (binding, first failing test, reason) of the row/col spaces and a sample of ld."""
    for sname in ("gemm_rowmajor", "gemm_colmajor"):
        _oracle_vs_golden(stem, sname)
    _oracle_vs_golden(stem, "gemm_rowmajor_ld", limit=1500)


@pytest.mark.parametrize("stem", CONV_STEMS)
def test_oracle_matches_reference_p2_conv(stem):
    _oracle_vs_golden(stem, "conv2d", limit=1200)


def test_oracle_cpu_xpu_gemm_agree():
    """profitability::sample_one's cross-check (profitability.cpp:76-85) holds for the restatements."""
    m, n, k = 24, 40, 56
    a = np.array([0.25 + (i % 17) * 0.0625 for i in range(m * k)], dtype=np.float32)
    b = np.array([-0.5 + (i % 23) * 0.0625 for i in range(k * n)], dtype=np.float32)
    c1 = O.cpu_gemm(a, b, m, n, k)
    c2 = O.xpu_gemm(a, b, m, n, k, threads=4)
    assert np.all(np.abs(c1.astype(np.float64) - c2) <= 1e-3 * (1 + np.abs(c1.astype(np.float64))))
