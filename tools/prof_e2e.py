"""Where the e2e step's time goes (prepared-sweep path, as in bench.py): host time
of the 35 atc_testsets_update_seeded calls, their GPU completion, the sweep replay
alone, and the two back to back."""
import ctypes as C
import dataclasses
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import torch

from paper_2301_11659_b200 import _lib, workloads
from paper_2301_11659_b200.evaluator import Evaluator, _TestsetHandle

ctx = _lib.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
L = _lib.lib()
_lib.check(ctx.handle, L.atc_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
ev = Evaluator(ctx)
jobs = workloads.corpus_jobs()
jobs.sort(key=lambda j: j.spec.semantics != "conv2d")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
progs = {}
for j in jobs:
    if j.stem in progs:
        continue
    s, keep = j.ts.seeded_struct(needed_only=True)
    keep = [pin(a) for a in keep]
    (s.int_values, s.ptr_is_f32, s.region_len, s.test_ok, s.stream_seed, s.stream_skip, s.diff_off, s.diff_pos,
     s.diff_val) = [a.ctypes.data for a in keep]
    out = C.c_void_p()
    _lib.check(ctx.handle, L.atc_testsets_upload_seeded(ctx.handle, C.byref(s), C.byref(out)))
    h = _TestsetHandle(ctx, out.value)
    progs[j.stem] = (s, keep, h, dataclasses.replace(j.ts, _handles={id(ctx): h}))
sweep = ev.sweep([(j.spec, progs[j.stem][3], j.space, 0, j.space.count) for j in jobs])


vals = list(progs.values())
structs = (_lib.SeededTestsets * len(vals))(*[v[0] for v in vals])
hptrs = (C.c_void_p * len(vals))(*[v[2].value for v in vals])


def updates():
    _lib.check(ctx.handle, L.atc_testsets_update_seeded_many(ctx.handle, hptrs, structs, len(vals)))


def timed(fn, reps=5):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        t0 = time.perf_counter()
        e0.record(stream)
        fn()
        th = time.perf_counter() - t0
        e1.record(stream)
        torch.cuda.synchronize()
        tw = time.perf_counter() - t0
        out.append((e0.elapsed_time(e1), th * 1e3, tw * 1e3))
    return np.median(np.array(out), axis=0)


for _ in range(3):
    updates()
    sweep.run()
for name, fn in (("updates", updates), ("sweep", sweep.run), ("both", lambda: (updates(), sweep.run()))):
    ev_ms, host_ms, wall_ms = timed(fn)
    print(f"{name:8s} events {ev_ms:.3f} ms  host enqueue {host_ms:.3f} ms  wall {wall_ms:.3f} ms")

# kernel timeline of one e2e step (CUPTI via torch.profiler): when the probe-image
# regeneration ends and the sweep's kernels start
import json as _json  # noqa: E402

from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        updates()
        sweep.run()
        torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/atc_e2e_trace.json")
evs = _json.load(open("/tmp/atc_e2e_trace.json"))["traceEvents"]
ks = sorted([e for e in evs if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
half = len(ks) // 2
ks = ks[half:]  # the second step
t0 = ks[0]["ts"]
from collections import defaultdict  # noqa: E402

agg = defaultdict(lambda: [0, 0.0, 1e18, 0.0])
for e in ks:
    a = agg[e["name"].split("(")[0][:40]]
    a[0] += 1
    a[1] += e["dur"]
    a[2] = min(a[2], e["ts"] - t0)
    a[3] = max(a[3], e["ts"] + e["dur"] - t0)
print(f"e2e step span {max(e['ts'] + e['dur'] for e in ks) - t0:.1f} us, {len(ks)} GPU ops")
for name, (n, dur, first, last) in sorted(agg.items(), key=lambda kv: kv[1][2]):
    print(f"{name:42s} n={n:3d} sum={dur:8.1f} us  first={first:8.1f}  last_end={last:8.1f}")
