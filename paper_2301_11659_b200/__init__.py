"""B200-native candidate-evaluation stage and API backends for ATC (arXiv 2301.11659).

The product is libatc_b200.so (C ABI: include/atc_b200.h) — hand-written sm_100a
CUDA kernels for the batched binding evaluator and the tcgen05 sgemm/conv2d
backends.  This package is the host-side mirror of the reference's interfaces
for that path (verify_rewrite, run_reference, the dispatch handler, cpu_gemm /
xpu_gemm) and the plumbing around it.  There is no CPU fallback: every compute
entry point raises AtcError if the CUDA library or an sm_100 device is missing.
"""
from ._lib import AtcError, Context, default_context, lib  # noqa: F401
from .evaluator import (BatchVerdicts, BindingSpace, Evaluator, RecordedTestsets,  # noqa: F401
                        record_testsets, verify_rewrite_batch)
from .spec import ApiSpec, SpecError, parse_api_spec  # noqa: F401
