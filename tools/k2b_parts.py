"""The corpus sweep (graph replay, CUDA events, median of 9) with the conv K2b's
(binding, t) items split over 1 / 2 / 4 / 8 warps (ATC_OPT_K2B_PARTS); every
variant's passing sets and histograms are checked equal."""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
import numpy as np
import torch

from paper_2301_11659_b200 import _lib, workloads
from paper_2301_11659_b200.evaluator import Evaluator

jobs = workloads.corpus_jobs()
jobs.sort(key=lambda j: j.spec.semantics != "conv2d")
out, ref = {}, None
for parts in (1, 2, 4, 8, 1):
    ctx = _lib.Context(0)
    ctx.set_option(_lib.OPT_K2B_PARTS, parts)
    stream = torch.cuda.Stream()
    _lib.check(ctx.handle, _lib.lib().atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
    ev = Evaluator(ctx)
    sw = ev.sweep([(j.spec, j.ts, j.space, 0, j.count) for j in jobs])
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
    got = [(r[0].tolist(), r[1], r[2].tolist()) for r in res]
    if ref is None:
        ref = got
    assert got == ref, parts
    out[f"parts{parts}"] = float(np.median(ts))
    print(parts, out[f"parts{parts}"], flush=True)
print(json.dumps(out))
