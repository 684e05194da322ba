"""Config 1 alone (naive_f32 at 64^3, both dense specs, T=16) as a prepared sweep: eager
runs (for an ncu launch list) then the graph-replayed time."""
import ctypes as C
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2301_11659_b200 import _lib, workloads  # noqa: E402
from paper_2301_11659_b200.evaluator import Evaluator  # noqa: E402

ctx = _lib.Context(0)
stream = torch.cuda.Stream()
_lib.check(ctx.handle, _lib.lib().atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
ev = Evaluator(ctx)
jobs = workloads.naive64_jobs()
sw = ev.sweep([(j.spec, j.ts, j.space, 0, j.space.count) for j in jobs])
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
print(sorted(ts)[3])
