"""One conv space (default conv_direct x conv2d) evaluated twice eagerly: the
launch list of the second run under `ncu --metrics gpu__time_duration.sum` is the
per-kernel chain of one space (tables, K1, K2-pre, K2a, K2b, finalize)."""
import sys

sys.path.insert(0, '.')
from paper_2301_11659_b200 import Evaluator, fixtures  # noqa: E402

stem = sys.argv[1] if len(sys.argv) > 1 else "conv_direct"
ev = Evaluator()
p = fixtures.load(stem)
ts = p.testsets(16)
sp = p.space("conv2d")
for _ in range(2):
    r = ev.eval_enumerated(fixtures.spec("conv2d"), ts, sp)
print(stem, r[1], r[2])
