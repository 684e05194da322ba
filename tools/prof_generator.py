"""k_probe_regions alone: atc_testsets_upload_seeded of one corpus program's test sets
(needed_only), timed with CUDA events over 10 uploads; under ncu the launches are
k_probe_regions (T CTAs, one per test)."""
import sys
import time

sys.path.insert(0, '.')
import torch

from paper_2301_11659_b200 import _lib, workloads

stem = sys.argv[1] if len(sys.argv) > 1 else "conv_direct"
ctx = _lib.Context(0)
j = next(j for j in workloads.corpus_jobs() if j.stem == stem)
for _ in range(3):
    h = j.ts.upload_seeded(ctx, needed_only=True)
    torch.cuda.synchronize()
    h.free()
ts = []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = j.ts.upload_seeded(ctx, needed_only=True)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
    h.free()
print(stem, "upload_seeded wall ms (median of 10):", sorted(ts)[5])
