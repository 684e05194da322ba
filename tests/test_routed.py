"""Routed dispatch host logic (rewriter.cpp:183-213) on CPU: the backend predictor
pinned to the reference's own train_svm model and predictions
(tests/golden/svm_volume.json, made by `python oracle/gen_golden.py --svm`), and the
predictor features of a call (rewriter.cpp:194-205)."""
import json
import os

from paper_2301_11659_b200 import backends, fixtures

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "svm_volume.json")


def test_svm_decision_matches_reference():
    g = json.load(open(GOLDEN))
    model = g["model"]
    predict = backends.svm_predictor(model)
    assert len(g["cases"]) > 1000
    for c in g["cases"]:
        d = backends.svm_decision(model, c["mnk"])
        assert abs(d - c["decision"]) <= 1e-9 * (1 + abs(c["decision"])), c
        assert predict(c["mnk"]) == c["backend"], c
    # rewriter_test.cpp:131-136: 2x2x2 routes to the host
    assert predict([2, 2, 2]) == 0


def test_routed_features():
    gemm, conv = fixtures.spec("gemm_rowmajor_ld"), fixtures.spec("conv2d")
    assert backends.routed_sizes(gemm, {"tc_m": 5, "tc_n": 6, "tc_k": 7, "tc_lda": 9}) == [5, 6, 7]
    sz = {"tc_n": 2, "tc_c": 3, "tc_h": 9, "tc_w": 8, "tc_k": 4, "tc_r": 3, "tc_s": 2, "tc_oh": 7, "tc_ow": 7}
    assert backends.routed_sizes(conv, sz) == [4, 2 * 7 * 7, 3 * 3 * 2]
    assert backends.routed_sizes(gemm, {}) == [1, 1, 1]  # role_size's default (rewriter.cpp:171)


def test_routed_labels_without_model():
    """rewriter_test.cpp:142-147: no model -> every call labelled "cpu"."""
    spec = fixtures.spec("gemm_rowmajor")
    choices = []
    h = backends.make_routed_dispatch(spec, None, choices)
    D = backends.DispatchArg
    try:  # the label is recorded before run_dispatch's checks (rewriter.cpp:190-210)
        h("atc_dispatch_gemm", [D("ptr", "a")], {})
    except RuntimeError as e:
        assert "arity" in str(e)
    assert choices == ["cpu"]
