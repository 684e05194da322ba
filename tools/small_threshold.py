"""Small-space sweep threshold A/B (ATC_OPT_SMALL_LOG2): config 1 (naive_f32 at 64^3,
both dense specs), config 4 (naive_ld x gemm_rowmajor_ld alone) and the corpus sweep,
graph-replayed, CUDA events, median of 9; results checked equal across settings."""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2301_11659_b200 import _lib, workloads  # noqa: E402
from paper_2301_11659_b200.evaluator import Evaluator  # noqa: E402

sets = {"config1": workloads.naive64_jobs(), "config4": workloads.stress_jobs(), "corpus": workloads.corpus_jobs()}
out, ref = {}, {}
for lg in (0, 12, 16, 20):
    ctx = _lib.Context(0)
    ctx.set_option(_lib.OPT_SMALL_LOG2, lg)
    stream = torch.cuda.Stream()
    _lib.check(ctx.handle, _lib.lib().atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
    ev = Evaluator(ctx)
    for name, js in sets.items():
        sw = ev.sweep([(j.spec, j.ts, j.space, 0, j.space.count) for j in js])
        for _ in range(3):
            res = sw.run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(9):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(stream)
            res = sw.run()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        sw.close()
        got = [(p.tolist(), n, h.tolist()) for p, n, h in res]
        ref.setdefault(name, got)
        assert got == ref[name], (name, lg)
        out[f"{name}_log2_{lg}"] = sorted(ts)[4]
    ctx.close()
print(json.dumps(out))
