"""Conv-space parity pinned beyond samples.  The conv spaces
(2.3e9 / 9.3e9 bindings) cannot be swept by the reference; tests/golden holds the
GPU's full passing lists (conv_passing.json) and the reference's own verify_rewrite
verdicts on the +-4096 neighbourhood of every passing index and pruned candidate
(conv_neighbourhoods.npz, oracle/gen_neighbourhoods.py).  CPU: the two fixtures
agree.  GPU: the per-binding path reproduces every neighbourhood verdict (first
failing test and reason) and a whole-space sweep returns exactly the pinned
passing lists at T = 16 and T = 10."""
import numpy as np
import pytest

from paper_2301_11659_b200 import Evaluator, fixtures, workloads


def test_neighbourhood_fixture_agrees_with_pinned_passing_sets():
    nb, passing = fixtures.conv_neighbourhoods(), fixtures.conv_passing()
    assert nb["radius"] >= 4096
    keys = [k for k in nb if k != "radius"]
    assert len(keys) == 8 and set(keys) == set(passing)
    total = 0
    for k in keys:
        v = nb[k]
        idx, reason, ft = v["idx"].astype(np.int64), v["reason"], v["fail_t"]
        total += len(idx)
        ref_pass = set(idx[reason == 0].tolist())
        inside = {p for p in passing[k]["16"]["passing"] if np.any(idx == p)}
        assert ref_pass == inside == set(passing[k]["16"]["passing"]), k
        assert set(passing[k]["16"]["passing"]) <= set(passing[k]["10"]["passing"])
        assert ((ft == -1) == (reason == 0)).all()
    assert total > 60000


@pytest.mark.gpu
def test_gpu_reproduces_reference_neighbourhood_verdicts():
    ev = Evaluator()
    nb = fixtures.conv_neighbourhoods()
    for k in [k for k in nb if k != "radius"]:
        stem, sname = k.rsplit("x", 1)
        p = fixtures.load(stem)
        space = p.space(sname)
        got = ev.eval_bindings(fixtures.spec(sname), p.testsets(16), *space.decode(nb[k]["idx"]))
        np.testing.assert_array_equal(got.fail_t, nb[k]["fail_t"], err_msg=k)
        np.testing.assert_array_equal(got.reason, nb[k]["reason"], err_msg=k)


@pytest.mark.gpu
@pytest.mark.parametrize("T", [16, 10])
def test_gpu_conv_sweep_equals_pinned_passing_sets(T):
    ev = Evaluator()
    pinned = fixtures.conv_passing()
    jobs = workloads.corpus_jobs(T, ("conv",))
    res = ev.eval_enumerated_many([(j.spec, j.ts, j.space, 0, j.count) for j in jobs], cap=1 << 16)
    for j, (pl, n, hist) in zip(jobs, res):
        assert pl.tolist() == pinned[f"{j.stem}x{j.spec_name}"][str(T)]["passing"]
        assert int(hist.sum()) == j.count and n == len(pl)
