"""Accepted-binding parity at pipeline level (pipeline.cpp:227-312).

For every GEMM/conv corpus program, the candidate loop with the batched P2
screen (GPU, or the reference's own P2 verdicts on CPU) plus host P1 on the
survivors must reproduce the reference pipeline's outcome from tests/golden/
pipeline.json: status, winning spec, winner rank and the accepted binding."""
import numpy as np
import pytest

from paper_2301_11659_b200 import fixtures
from paper_2301_11659_b200.pipeline import SpecCandidates, lift_function

SPEC_ORDER = ["gemm_rowmajor", "gemm_colmajor", "gemm_rowmajor_ld", "conv2d"]  # tools/liftc.cpp:60
P1_NAMES = {0: "Equivalent", 1: "NotEquivalent", 2: "Inconclusive"}


def _reference_outcome(stem):
    p = fixtures.load(stem)
    for rep in fixtures.pipeline_reports():
        if rep["file"] != p.meta["file"]:
            continue
        for f in rep["functions"]:
            if f["function"] == p.function:
                return f
    raise KeyError(stem)


def _cases():
    out = []
    for stem in fixtures.stems():
        p = fixtures.load(stem)
        if "specs" not in p.meta:
            continue
        ref = _reference_outcome(stem)
        if ref["status"] == "Misclassified":
            continue
        out.append(stem)
    return out


def _run(stem, p2_override=None, evaluator=None):
    p = fixtures.load(stem)
    ref = _reference_outcome(stem)
    label = "gemm" if p.meta["corpus_dir"] == "gemm" else "conv2d"
    specs, p1_table = [], {}
    for sname in SPEC_ORDER:
        spec = fixtures.spec(sname)
        if spec.semantics != label:
            continue
        s = p.meta["specs"][sname]
        ranked = [{"arrays": c["arrays"], "sizes": c["sizes"], "scalars": c["scalars"]} for c in s["pruned"]]
        for c in s["pruned"]:
            p1_table[(sname, str(sorted(c["arrays"].items())), str(sorted(c["sizes"].items())))] = P1_NAMES[c["p1"]]
        specs.append(SpecCandidates(spec, ranked, s["truncated"]))

    def p1(spec, cand):
        return p1_table[(spec.name, str(sorted(cand["arrays"].items())), str(sorted(cand["sizes"].items())))]

    out = lift_function(specs, p.testsets(10), p.user_ptrs, p1, evaluator=evaluator, p2_override=p2_override)
    assert out.status == ref["status"], (stem, out.status, ref["status"])
    if ref["status"] == "Lifted":
        man = ref["manifest"]
        assert out.winning_api == ref["winning_api"]
        assert out.winner_rank == man["candidates"]["winner_rank"]
        assert out.binding["arrays"] == man["binding"]["arrays"]
        assert out.binding["sizes"] == man["binding"]["sizes"]
    return out


def _golden_p2(stem):
    p = fixtures.load(stem)

    def p2(spec, am, sm):
        v = p.verdicts(spec.name)
        space = p.space(spec.name)
        idx = [space.index_of({"arrays": {a: p.user_ptrs[am[b, i]] for i, a in enumerate(space.api_arrays)},
                               "sizes": {a: p.user_ints[sm[b, q]] for q, a in enumerate(space.api_sizes)}})
               for b in range(am.shape[0])]
        pos = {int(g): i for i, g in enumerate(v["idx"])}
        ft = np.array([v["fail_t"][pos[g]] for g in idx])
        return (ft < 0) | (ft >= 10)

    return p2


@pytest.mark.parametrize("stem", _cases())
def test_pipeline_outcome_with_reference_p2(stem):
    """Host logic only: the reference's own P2 verdicts through lift_function."""
    _run(stem, p2_override=_golden_p2(stem))


@pytest.mark.gpu
@pytest.mark.parametrize("stem", _cases())
def test_pipeline_outcome_with_gpu_p2(stem):
    """The batched GPU P2 screen + host P1 reproduce the reference pipeline's
    accepted binding (all 26 GEMM + 8 conv programs)."""
    out = _run(stem)
    # the GPU screen leaves the host at most a couple of P1 calls per program
    assert out.p1_calls <= 3
