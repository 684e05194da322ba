"""Helper for tests/test_gpu_eval.py::test_conv_screen_kernels_agree: evaluates a
few conv spaces/ranges/test-set variants and prints the results as JSON, so the
test can run it under ATC_SCREEN_PLANES=1 / ATC_SCREEN_GENERIC=1 (read once per
process by libatc_b200) and compare the three K1 conv kernels."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2301_11659_b200 import Evaluator, fixtures  # noqa: E402
from tests.test_gpu_eval import CONV_VARIANTS  # noqa: E402

CASES = [("conv_direct", "in_700_out_900", 0, 1 << 21), ("conv_permuted_sig", "wt_200", 1234567, 1234567 + 999_999),
         ("im2col_buffered", "recorded", 0, None), ("conv_direct", "zero_int", 17, 2_000_017),
         ("winograd_1d", "in_3000", 5_000_000, 9_000_000)]


def main():
    ev = Evaluator()
    out = []
    for stem, variant, b, e in CASES:
        p = fixtures.load(stem)
        space = p.space("conv2d")
        ts = CONV_VARIANTS[variant](p.testsets(16))
        passing, n, hist = ev.eval_enumerated(fixtures.spec("conv2d"), ts, space, b, space.count if e is None else e)
        out.append({"case": [stem, variant, b, e], "passing": passing.tolist(), "n": n, "hist": hist.tolist()})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
