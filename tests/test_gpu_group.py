"""Device groups (atc_group_*) on the GPU box: a one-device group
and a group listing device 0 twice (two independent contexts on one B200 — the
shard plan, the per-member evaluation and the combine are exercised exactly as
with two GPUs; no kernel waits on another member) return, for every job, the
passing set, reason histogram and first passing index of the single-context
evaluator (itself pinned to the reference's verdicts by test_gpu_eval.py)."""
import numpy as np
import pytest

from paper_2301_11659_b200 import Evaluator, fixtures
from paper_2301_11659_b200 import _lib as L
from paper_2301_11659_b200.group import Group

pytestmark = pytest.mark.gpu

ITEMS = [("naive_ld", "gemm_rowmajor_ld", 0, None), ("conv_direct", "conv2d", 381367044 - (1 << 22), 381367044 + (1 << 22)),
         ("naive_rowmajor", "gemm_colmajor", 0, None), ("winograd_1d", "conv2d", 0, 1 << 25),
         ("vec8_unguarded", "gemm_rowmajor", 0, None), ("conv3x3_unrolled", "conv2d", 380835603 - 5, 381426093 + 5)]


def _items(T=16):
    out = []
    for stem, sname, b, e in ITEMS:
        p = fixtures.load(stem)
        space = p.space(sname)
        out.append((fixtures.spec(sname), p.testsets(T), space, b, space.count if e is None else e))
    return out


@pytest.fixture(scope="module")
def single():
    ev = Evaluator()
    return [ev.eval_enumerated(spec, ts, space, b, e) for spec, ts, space, b, e in _items()]


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_group_matches_single_context(single, devices):
    g = Group(devices)
    assert g.size == len(devices)
    items = _items()
    for run in (g.eval_enumerated_many(items), g.sweep(items).run()):
        for (pg, ng, hg, first), (ps, ns, hs) in zip(run, single):
            np.testing.assert_array_equal(pg, ps)
            assert ng == ns and hg.tolist() == hs.tolist()
            assert first == (int(ps[0]) if ns else -1)
    g.close()


def test_group_prepared_sweep_replays(single):
    """A prepared group sweep (one CUDA graph per member after the first run) gives
    the same results on every replay."""
    g = Group([0, 0])
    sw = g.sweep(_items())
    for _ in range(3):
        for (pg, ng, hg, first), (ps, ns, hs) in zip(sw.run(), single):
            np.testing.assert_array_equal(pg, ps)
            assert ng == ns and hg.tolist() == hs.tolist()
    sw.close()
    g.close()


def test_group_members_are_usable_contexts():
    """Each member is an ordinary context (one per pipeline worker thread)."""
    g = Group([0, 0])
    p = fixtures.load("naive_rowmajor")
    spec, space = fixtures.spec("gemm_rowmajor"), p.space("gemm_rowmajor")
    am, sm = space.decode(np.arange(space.count))
    firsts = [Evaluator(g.member(i)).eval_bindings(spec, p.testsets(10), am, sm).first_pass for i in range(2)]
    assert firsts == [21, 21]
    g.close()


def test_group_rejects_bad_device():
    with pytest.raises(L.AtcError):
        Group([0, 97])
