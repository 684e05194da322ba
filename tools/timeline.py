"""Kernel timeline of one graph-replayed corpus sweep step (torch.profiler / CUPTI):
per kernel its stream, start and end relative to the step's first kernel, and per
stream the busy time — which chain is the critical path of the concurrent step.

    python tools/timeline.py [--steps N] [--json OUT]
"""
import argparse
import ctypes as C
import json
import sys
from collections import defaultdict

sys.path.insert(0, '.')
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2301_11659_b200 import _lib, workloads
from paper_2301_11659_b200.evaluator import Evaluator

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--json", default=None)
ap.add_argument("--only", default=None, help="STEM:SPEC — one space's chain")
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
for _ in range(4):
    sw.run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(args.steps):
        sw.run()
        torch.cuda.synchronize()
sw.close()
trace = "/tmp/atc_timeline.json"
prof.export_chrome_trace(trace)
with open(trace) as f:
    evs = [e for e in json.load(f)["traceEvents"] if e.get("cat") == "kernel"]
evs.sort(key=lambda e: e["ts"])
# split into steps at gaps > 50 us
steps, cur = [], []
for e in evs:
    if cur and e["ts"] - max(x["ts"] + x["dur"] for x in cur) > 50:
        steps.append(cur)
        cur = []
    cur.append(e)
if cur:
    steps.append(cur)
st = steps[-1]
t0 = st[0]["ts"]
span = max(e["ts"] + e["dur"] for e in st) - t0
rows = [{"kernel": e["name"].split("(")[0][:40], "stream": e["args"].get("stream"), "start_us": round(e["ts"] - t0, 1),
         "dur_us": round(e["dur"], 1)} for e in st]
busy = defaultdict(float)
for r in rows:
    busy[r["stream"]] += r["dur_us"]
out = {"step_span_us": round(span, 1), "kernels": len(rows), "stream_busy_us": dict(busy), "timeline": rows}
for r in rows:
    print(f'{r["start_us"]:8.1f} {r["start_us"] + r["dur_us"]:8.1f}  s{r["stream"]:<4} {r["kernel"]}')
print(json.dumps({k: v for k, v in out.items() if k != "timeline"}))
if args.json:
    with open(args.json, "w") as f:
        json.dump(out, f, indent=1)
