"""Corpus sweep split by class (--fp32: ATC_MODE_FP32_SCREEN): conv-only and gemm-only sweeps timed alone (CUDA
events, graph replay), then one conv-only sweep per job for the per-space cost.
Under ncu (`--metrics gpu__time_duration.sum`) the last eager run of each sweep
gives the per-kernel launch list."""
import ctypes as C
import sys

sys.path.insert(0, '.')
import torch

from paper_2301_11659_b200 import _lib, workloads
from paper_2301_11659_b200.evaluator import Evaluator

ctx = _lib.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
_lib.check(ctx.handle, _lib.lib().atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
ev = Evaluator(ctx)
jobs = workloads.corpus_jobs()


MODE = _lib.MODE_FP32_SCREEN if "--fp32" in sys.argv else _lib.MODE_FP64


def timed(items, reps=5):
    sw = ev.sweep(items, mode=MODE)
    for _ in range(3):
        sw.run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        sw.run()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    sw.close()
    return sorted(ts)[reps // 2]


conv = [j for j in jobs if j.spec.semantics == "conv2d"]
gemm = [j for j in jobs if j.spec.semantics != "conv2d"]
full = lambda js: [(j.spec, j.ts, j.space, 0, j.space.count) for j in js]  # noqa: E731
print(f"all {timed(full(conv + gemm)):.3f} ms  conv-only {timed(full(conv)):.3f} ms  gemm-only {timed(full(gemm)):.3f} ms")
for j in conv:
    print(f"  {j.stem + " x " + j.spec_name:40s} {j.space.count:>14,d} bindings  {timed(full([j])):.3f} ms")
