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
base = None
for world in (1, 2, 4, 8):
    worst, per = 0, []
    for rank in range(world):
        sh = workloads.plan_shards(jobs, rank, world)
        sw = ev.sweep([(j.spec, j.ts, j.space, b, e) for j, (b, e) in zip(jobs, sh)])
        for _ in range(3): sw.run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(stream); sw.run(); e1.record(stream); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        per.append(sorted(ts)[2]); worst = max(worst, per[-1]); sw.close()
    base = base or worst
    print(f"world {world}: slowest rank's sweep {worst:.2f} ms (ranks: {' '.join(f'{x:.2f}' for x in per)}), "
          f"ideal {base / world:.2f}")
