import sys, ctypes as C
sys.path.insert(0, '.')
import torch
from paper_2301_11659_b200 import workloads, _lib
from paper_2301_11659_b200.evaluator import Evaluator
ctx = _lib.Context(0)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
_lib.check(ctx.handle, _lib.lib().atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
ev = Evaluator(ctx)
jobs = workloads.corpus_jobs(); jobs.sort(key=lambda j: j.spec.semantics != "conv2d")
def timed(items):
    sw = ev.sweep(items)
    for _ in range(3): sw.run()
    torch.cuda.synchronize(); ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream); sw.run(); e1.record(stream); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    sw.close(); return sorted(ts)[2]
for world, rank in ((8, 0), (8, 3), (8, 7)):
    sh = workloads.plan_shards(jobs, rank, world)
    items = [(j.spec, j.ts, j.space, b, e) for j, (b, e) in zip(jobs, sh) if e > b]
    conv = [it for it in items if it[0].semantics == "conv2d"]
    gemm = [it for it in items if it[0].semantics != "conv2d"]
    print(world, rank, f"all {timed(items):.3f} conv {timed(conv):.3f} ({len(conv)}: {[ (it[2].count, it[4]-it[3]) for it in conv]}) gemm {timed(gemm):.3f} ({len(gemm)})")
    for it in conv: print("   ", it[2].count, it[4]-it[3], f"{timed([it]):.3f}")
