"""The ResNet-50 unit-stride conv layers of bench.py (N=256, TF32) through
atc_conv2d_nchw_device against cuDNN (torch conv2d, TF32, benchmark mode): CUDA events
over 20 calls each, optionally under context tc flags (argv[1], ATC_OPT_TC_FLAGS)."""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
import torch

from bench import RESNET_LAYERS
from paper_2301_11659_b200 import _lib

flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
ctx = _lib.Context(0)
if flags:
    ctx.set_option(_lib.OPT_TC_FLAGS, flags)
L = _lib.lib()
s = torch.cuda.Stream()
torch.backends.cudnn.benchmark = True
torch.backends.cudnn.allow_tf32 = True


def timed(fn, reps=20):
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = []
for name, c, k, r, h in RESNET_LAYERS:
    n, oh = 256, h - r + 1
    x = torch.empty(n, c, h, h, device="cuda").uniform_(-1, 1)
    w = torch.empty(k, c, r, r, device="cuda").uniform_(-1, 1)
    y = torch.empty(n, k, oh, oh, device="cuda")

    def run():
        _lib.check(ctx.handle, L.atc_conv2d_nchw_device(ctx.handle, x.data_ptr(), w.data_ptr(), y.data_ptr(), n, c, h,
                                                        h, k, r, r, _lib.PREC_TF32, C.c_void_p(s.cuda_stream)))

    ms = timed(run)
    ref = torch.nn.functional.conv2d(x, w)
    err = ((y - ref).abs().max() / ref.abs().max()).item()  # every image
    ms_lib = timed(lambda: torch.nn.functional.conv2d(x, w))
    fl = 2 * n * k * oh * oh * c * r * r
    out.append({"layer": name, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1),
                "cudnn_tflops": round(fl / ms_lib / 1e9, 1), "ratio": round(ms_lib / ms, 3), "err_vs_cudnn": err})
    print(json.dumps(out[-1]))
