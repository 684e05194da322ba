"""Host-side checks that need no GPU: the C ABI library loads and exports every
symbol include/atc_b200.h declares; spec decode tables; golden-data invariants
 the GPU tests rely on."""
import os
import re

import numpy as np
import pytest

from paper_2301_11659_b200 import _lib, fixtures
from paper_2301_11659_b200.probe import Rng, SizeRules, draw_sizes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    with open(os.path.join(ROOT, "include", "atc_b200.h")) as f:
        text = f.read()
    declared = set(re.findall(r"\b(atc_[a-z0-9_]+)\s*\(", text))
    assert declared, "no declarations parsed"
    lib = _lib.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), f"libatc_b200.so does not export {name}"
    assert declared == set(_lib.EXPORTED), sorted(declared ^ set(_lib.EXPORTED))


def test_no_device_here_fails_loudly():
    """No CUDA device in this container: creating a context must raise, never fall back."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert _lib.lib().atc_device_count() == 0
    with pytest.raises(_lib.AtcError):
        _lib.Context(0)


def test_spec_decode_tables():
    d = fixtures.spec("gemm_rowmajor_ld").to_desc()
    assert (d.semantics, d.layout, d.n_arrays, d.n_sizes) == (0, 0, 3, 6)
    assert [d.array_role[a] for a in range(3)] == [0, 1, 2]
    assert [d.array_livein[a] for a in range(3)] == [1, 1, 0]
    assert list(d.array_dims[0])[:2] == [0, 3]  # A dims (m, lda), canonical order
    assert [d.role_size[r] for r in range(6)] == [0, 1, 2, 3, 4, 5]
    c = fixtures.spec("conv2d").to_desc()
    assert c.semantics == 1 and c.n_sizes == 9
    assert [c.role_size[6 + r] for r in range(9)] == list(range(9))
    assert [c.role_size[r] for r in range(6)] == [-1] * 6


def test_draw_sizes_rules():
    """analysis.cpp:25-71 with multiple_of rounding and derived rules."""
    rules = SizeRules.from_json({"ranges": {"m": [5, 9]}, "multiple_of": {"m": 4},
                                 "derived": {"oh": {"terms": [[1, "h"], [-1, "r"]], "constant": 1}}})
    for seed in range(50):
        s = draw_sizes(["m", "h", "r", "oh"], rules, Rng(seed))
        assert s is None or (s["m"] == 8 and s["oh"] == s["h"] - s["r"] + 1)
        if s is None:  # only when the derived oh lands below 1
            pass


def _p2_pass_set(stem, sname, T=10):
    p = fixtures.load(stem)
    v = p.verdicts(sname)
    ok = (v["fail_t"] < 0) | (v["fail_t"] >= T)
    return v["idx"][ok].tolist()


def test_appendix_a_accepted_sets():
    """SURVEY.md Appendix A, from the reference dump (T=10): P2-passing indices, and
    P1 agrees except gemm_square (P2 not a subset of P1)."""
    expect = {("naive_rowmajor", "gemm_rowmajor"): [21], ("naive_rowmajor", "gemm_colmajor"): [73],
              ("naive_colmajor", "gemm_rowmajor"): [73], ("naive_colmajor", "gemm_colmajor"): [21],
              ("strassen_staged", "gemm_rowmajor"): [21, 48], ("strassen_staged", "gemm_colmajor"): [181, 208],
              ("blocked_copy_local", "gemm_rowmajor"): [21], ("blocked_copy_local", "gemm_colmajor"): [181],
              ("naive_ld", "gemm_rowmajor_ld"): [44790], ("naive_ld", "gemm_rowmajor"): [],
              ("accum_inplace", "gemm_rowmajor"): [], ("vec8_unguarded", "gemm_colmajor"): [],
              ("gemm_square", "gemm_rowmajor"): [0]}
    for (stem, sname), want in expect.items():
        assert _p2_pass_set(stem, sname) == want, (stem, sname)
        p = fixtures.load(stem)
        v = p.verdicts(sname)
        p1_eq = v["idx"][v["p1"] == 0].tolist()
        assert p1_eq == ([] if stem == "gemm_square" else want), (stem, sname, p1_eq)


def test_pipeline_golden_statuses():
    """The reference pipeline's corpus outcome: every status
    agrees with the sidecar's expect_lift."""
    reps = fixtures.pipeline_reports()
    lifted = {r["file"] for r in reps for f in r["functions"]
              if f["function"] == r["function_of_interest"] and f["status"] == "Lifted"}
    for r in reps:
        if r["function_of_interest"]:
            assert (r["file"] in lifted) == bool(r["expect_lift"]), r["file"]
    assert len([f for f in lifted if f.startswith(("conv", "im2col", "winograd"))]) == 6


def test_binding_space_decode_roundtrip():
    p = fixtures.load("conv_direct")
    space = p.space("conv2d")
    assert space.count == 2324522934
    idx = np.array([0, 1, 12345678901 % space.count, space.count - 1], dtype=np.uint64)
    am, sm = space.decode(idx)
    for i, g in enumerate(idx):
        b = space.binding(int(g))
        assert space.index_of(b) == int(g)
        assert [space.user_ptrs[x] for x in am[i]] == [b["arrays"][a] for a in space.api_arrays]
