"""The reference-side adapter (integration/atc_liftc_adapter.cpp), compiled against
the unmodified reference into oracle/_ref/adapter_check, driving libatc_b200 from the
reference's own C++ (test infrastructure: it links the oracle build)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "oracle", "_ref", "adapter_check")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(TOOL), reason="oracle/_ref/adapter_check not built")]


def _run(*args, timeout=900):
    r = subprocess.run([TOOL, *args], capture_output=True, text=True, timeout=timeout)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    return r.returncode, lines, r.stderr


def test_adapter_reproduces_reference_pipeline():
    """Reference lift_program vs the adapter's candidate_loop (analysis + matching +
    ranking unchanged, one prefix upload + one GPU P2 batch for every spec, host P1
    in rank order): the masked report_to_json of every corpus function is
    byte-identical — status, status_detail, by_spec, evaluated[] verdicts AND
    details (VerificationFailed details recomputed from the GPU's (t, reason)),
    winner and manifest — and the production setting (P1 only on P2 survivors)
    picks the same winner."""
    rc, lines, err = _run("corpus")
    assert rc == 0, err + json.dumps(lines[-3:])[:4000]
    assert lines[-1]["mismatches"] == 0
    # every function of all 55 corpus files (gemm, conv, nonidiom); 34 reach the
    # candidate stage (the rest are Misclassified: no candidate stage in either)
    assert len({x["stem"] for x in lines[:-1]}) == 55 and len(lines) - 1 == 58
    funcs = [x for x in lines[:-1] if x.get("candidate_stage")]
    assert len(funcs) == 34
    assert all(x["same_report_json"] and x["fast_same_winner"] for x in funcs)
    lifted = [x for x in funcs if x.get("gpu_status") == "Lifted"]
    assert len(lifted) == 29  # 23 GEMM + 6 conv


def test_adapter_p2_details_match_verify_rewrite():
    """A VerificationFailed entry's detail (pipeline.cpp:279-283) is rebuilt from the
    GPU's (first failing test, reason) — atc_dispatch on that test's recorded image,
    compared in the reference's order — and equals rewriter::verify_rewrite's own
    detail on P2-rejected bindings of every corpus program x spec."""
    rc, lines, err = _run("details", "24")
    assert rc == 0, err + json.dumps(lines[:5])[:4000]
    last = lines[-1]
    assert last["mismatches"] == 0 and last["checked"] > 1000
    # every corpus rejection is a mismatch: with 65,536-element probe regions and
    # sizes drawn in [2, 8] (or the sidecars' small ranges) no extent check of
    # run_dispatch (rewriter.cpp:136-148) can fail, so "dispatch failed" details
    # never arise on recorded corpus test sets (the dispatch messages themselves are
    # pinned by tests/test_gpu_backends.py)
    assert last["kinds"].get("mismatch", 0) == last["checked"]


def test_adapter_gpu_dispatch_bit_identical():
    """make_gpu_dispatch vs make_oracle_dispatch on every lifted corpus function."""
    rc, lines, err = _run("dispatch")
    assert rc == 0, err
    assert lines[-1]["mismatches"] == 0


def test_adapter_unpruned_stress_space():
    """naive_ld x gemm_rowmajor_ld (279,936 bindings): gpu::first_accepted_unpruned on
    the device group (every visible GPU; enumerated P2 sharded over the members, host
    P1 on the survivors) and the same space as one explicit ranked list on one context
    agree — the GPU screen leaves one survivor, host P1 accepts it (index 44790, the
    identity)."""
    rc, lines, err = _run("unpruned", "naive_ld", "gemm_rowmajor_ld", "10")
    assert rc == 0, err + json.dumps(lines)[:2000]
    j = lines[-1]
    assert j["bindings"] == 279936 and j["same"]
    for k in ("group", "list"):
        assert j[k]["p2_passed"] == 1 and j[k]["winner"] == 44790 and j[k]["p1_calls"] == 1


def test_adapter_unpruned_conv_space_on_group():
    """conv_direct x conv2d — all 2,324,522,934 bindings of the unpruned space through
    the adapter on the device group (no explicit list could hold it): P1 accepts the
    reference's pruned winner, the identity binding at index 381367044."""
    rc, lines, err = _run("unpruned", "conv_direct", "conv2d", "10")
    assert rc == 0, err + json.dumps(lines)[:2000]
    j = lines[-1]
    assert j["bindings"] == 2324522934 and j["same"] and "list" not in j
    g = j["group"]
    assert g["winner"] == 381367044 and g["p2_passed"] >= 1 and sum(g["reason_counts"]) == 2324522934


def test_adapter_routed_dispatch():
    """make_gpu_routed_dispatch vs rewriter::make_routed_dispatch (rewriter.cpp:183-213):
    identical cpu/xpu labels on every lifted corpus function, bit-identical results on
    the exact route; f32 GEMM (row/col/ld) and conv calls labelled "xpu" run on the
    tcgen05 backends within their stated TF32 / 3xTF32 bounds; "cpu" stays exact."""
    rc, lines, err = _run("routed")
    assert rc == 0, err + json.dumps([x for x in lines if not x.get("ok", True)][:3])
    assert lines[-1]["mismatches"] == 0
    direct = [x for x in lines if "direct" in x]
    assert len(direct) == 8 and all(x["ok"] for x in direct)


def test_adapter_b200_profitability_sampler():
    """profitability::sample_one / sample_timings (profitability.cpp:65-118) with the
    accelerator side on the B200 backend the routed dispatch calls (atc_sgemm_rm,
    host buffers in and out): every grid point passes the reference's cross-check
    against cpu_gemm, both labels occur, and the reference's own train_svm on these
    labels predicts the holdout grid (the model the routed "xpu" label comes from is
    trained on the backend it dispatches to)."""
    rc, lines, err = _run("sampler")
    assert rc == 0, err
    j = lines[-1]
    assert j["samples"] == 60 and 0 < j["xpu_labels"] < 60
    # the labels are wall-clock races (B200 through PCIe vs the host GEMM), so points near
    # the break-even size flip between runs: 0.90 / 0.85 and 0.85 / 0.85 both measured
    assert j["train_accuracy"] >= 0.8 and j["holdout_accuracy"] >= 0.75
