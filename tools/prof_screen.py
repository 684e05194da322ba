import sys, time, ctypes as C
sys.path.insert(0, '.')
import numpy as np
from paper_2301_11659_b200 import Evaluator, fixtures, _lib
ev = Evaluator()
L = _lib.lib()
for stem, sname in (("conv_direct", "conv2d"), ("im2col_buffered", "conv2d"), ("naive_ld", "gemm_rowmajor_ld")):
    p = fixtures.load(stem)
    ts = p.testsets(16)
    sp = p.space(sname)
    ev.eval_enumerated(fixtures.spec(sname), ts, sp, 0, min(sp.count, 1 << 26))
    prof = _lib.Profile()
    L.atc_profile_start(ev.ctx.handle)
    t0 = time.time()
    passing, cnt, hist = ev.eval_enumerated(fixtures.spec(sname), ts, sp)
    dt = time.time() - t0
    L.atc_profile_read(ev.ctx.handle, C.byref(prof))
    print(stem, sname, sp.count, f"wall {dt*1e3:.1f} ms", f"{sp.count/dt:.3e}/s", "screen_ms", round(prof.screen_ms, 2),
          "confirm_ms", round(prof.confirm_ms, 2), "survivors", prof.survivors, "pass", cnt, passing[:4], "hist", hist.tolist())
