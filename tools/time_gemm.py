"""sgemm TF32 8192^3 on a side stream, CUDA events over 20 launches (tcgen05 kernel vs
cuBLAS TF32 on the same operands)."""
import ctypes as C
import sys

sys.path.insert(0, '.')
import torch

from paper_2301_11659_b200 import _lib

ctx = _lib.Context(0)
if len(sys.argv) > 2:  # context tc flags (ATC_OPT_TC_FLAGS)
    ctx.set_option(_lib.OPT_TC_FLAGS, int(sys.argv[2]))
L = _lib.lib()
m = n = k = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.rand(m, k, device="cuda") * 2 - 1
b = torch.rand(k, n, device="cuda") * 2 - 1
c = torch.empty(m, n, device="cuda")
st = torch.cuda.Stream()


def run():
    _lib.check(ctx.handle, L.atc_sgemm_rm_device(ctx.handle, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, 0,
                                                 C.c_void_p(st.cuda_stream)))


def timed(fn, reps=20):
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = timed(run)
torch.backends.cuda.matmul.allow_tf32 = True
ms_cublas = timed(lambda: torch.matmul(a, b, out=c))
fl = 2 * m * n * k
print(f"tcgen05 {ms:.3f} ms {fl / ms / 1e9:.1f} TFLOP/s   cuBLAS {ms_cublas:.3f} ms {fl / ms_cublas / 1e9:.1f} TFLOP/s")
