"""The gemm spaces of the corpus as one prepared sweep (k_sweep_small): K1 survivors
(atc_profile), the graph-replayed time (CUDA events, median of 7) — and under ncu the
k_sweep_small launch of the eager runs."""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2301_11659_b200 import _lib, workloads  # noqa: E402
from paper_2301_11659_b200.evaluator import Evaluator  # noqa: E402

ctx = _lib.Context(0)
stream = torch.cuda.Stream()
_lib.check(ctx.handle, _lib.lib().atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
ev = Evaluator(ctx)
jobs = workloads.corpus_jobs(16, ("gemm",))
sw = ev.sweep([(j.spec, j.ts, j.space, 0, j.space.count) for j in jobs])
L = _lib.lib()
_lib.check(ctx.handle, L.atc_profile_start(ctx.handle))
sw.run()
prof = _lib.Profile()
_lib.check(ctx.handle, L.atc_profile_read(ctx.handle, C.byref(prof)))
for _ in range(3):
    sw.run()
torch.cuda.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(stream)
    sw.run()
    e1.record(stream)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"survivors": prof.survivors, "kernels": prof.kernels, "ms": sorted(ts)[3]}))
