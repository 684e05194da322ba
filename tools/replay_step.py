"""Graph-replayed corpus sweep steps under the CUDA profiler range, for ncu.

    python tools/replay_step.py [--steps N] [--only STEM:SPEC] [--flush]

Builds the bench's corpus sweep (or one space with --only), runs it eagerly and
captures it (warm-up, outside the profiler range), then replays it N times between
cudaProfilerStart/Stop.  With `ncu --profile-from-start off` only the replayed
steps are captured, e.g.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \\
        --csv --log-file profiles/r2_replay_launches.csv python tools/replay_step.py --steps 1
    ncu --profile-from-start off --set full --clock-control none --import-source on \\
        -k regex:k_screen_conv_pairs -c 1 -o k1 python tools/replay_step.py --only conv_direct:conv2d

and tools/launch_shares.py turns the launch list into per-kernel shares of a step.
"""
import argparse
import ctypes as C
import sys

sys.path.insert(0, '.')
import torch

from paper_2301_11659_b200 import _lib, workloads
from paper_2301_11659_b200.evaluator import Evaluator

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--only", default=None)
ap.add_argument("--flush", action="store_true", help="256 MB L2 flush before each step (as bench.py)")
args = ap.parse_args()

ctx = _lib.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
_lib.check(ctx.handle, _lib.lib().atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
ev = Evaluator(ctx)
jobs = workloads.corpus_jobs()
jobs.sort(key=lambda j: j.spec.semantics != "conv2d")
if args.only:
    stem, spec = args.only.split(":")
    jobs = [j for j in jobs if j.stem == stem and j.spec_name == spec]
sw = ev.sweep([(j.spec, j.ts, j.space, 0, j.count) for j in jobs])
for _ in range(3):  # eager, capture, replay
    sw.run()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
ms = []
for _ in range(args.steps):
    if args.flush:
        flush.fill_(1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.profiler.start()
    e0.record(stream)
    sw.run()
    e1.record(stream)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ms.append(e0.elapsed_time(e1))
sw.close()
print(f"replayed {args.steps} step(s) of {len(jobs)} spaces: {ms} ms")
