"""Per conv corpus space: bindings, K1 (screen) and K2 (confirm) milliseconds of one
eager evaluation (atc profile), survivors — which chains are long in a sweep."""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
from paper_2301_11659_b200 import Evaluator, _lib, workloads  # noqa: E402

ev = Evaluator()
L = _lib.lib()
out = []
for j in workloads.corpus_jobs():
    if j.spec.semantics != "conv2d":
        continue
    ev.eval_enumerated(j.spec, j.ts, j.space)
    prof = _lib.Profile()
    L.atc_profile_start(ev.ctx.handle)
    _, cnt, _ = ev.eval_enumerated(j.spec, j.ts, j.space)
    L.atc_profile_read(ev.ctx.handle, C.byref(prof))
    out.append({"space": f"{j.stem}x{j.spec_name}", "bindings": j.space.count, "perms": len(j.space.perms)
                if hasattr(j.space, "perms") else None, "screen_ms": round(prof.screen_ms, 3),
                "confirm_ms": round(prof.confirm_ms, 3), "survivors": prof.survivors, "passing": cnt})
    print(json.dumps(out[-1]), flush=True)
