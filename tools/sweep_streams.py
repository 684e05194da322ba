"""The corpus sweep (graph replay, CUDA events, median of 7) with the conv chains on
1..4 concurrent streams (atc_set_option ATC_OPT_CONV_STREAMS), plus the conv-only and
gemm-only (k_sweep_small) sweeps; every run's passing sets are checked equal."""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2301_11659_b200 import _lib, workloads  # noqa: E402
from paper_2301_11659_b200.evaluator import Evaluator  # noqa: E402

jobs = workloads.corpus_jobs()
full = lambda js: [(j.spec, j.ts, j.space, 0, j.space.count) for j in js]  # noqa: E731
out, ref = {}, None
for streams in (1, 2, 4, 6, 8):
    ctx = _lib.Context(0)
    ctx.set_option(_lib.OPT_CONV_STREAMS, streams)
    stream = torch.cuda.Stream()
    _lib.check(ctx.handle, _lib.lib().atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
    ev = Evaluator(ctx)
    for name, js in (("all", jobs), ("conv", [j for j in jobs if j.spec.semantics == "conv2d"]),
                     ("gemm", [j for j in jobs if j.spec.semantics != "conv2d"])):
        if streams > 1 and name == "gemm":
            continue
        sw = ev.sweep(full(js))
        for _ in range(3):
            res = sw.run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(stream)
            res = sw.run()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        sw.close()
        if name == "all":
            got = [(p.tolist(), n, h.tolist()) for p, n, h in res]
            ref = ref or got
            assert got == ref, f"streams={streams}: results differ"
        out[f"{name}_streams{streams}"] = sorted(ts)[3]
    ctx.close()
print(json.dumps(out))
