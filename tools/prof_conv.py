"""The ResNet-50 unit-stride conv layers of bench.py (N=256, TF32) through
atc_conv2d_nchw_device, each warmed up and then run once between
cudaProfilerStart/Stop — the launches the conv-backend ncu captures profile:

    ncu --profile-from-start off --set full --clock-control none -k regex:k_tc_gemm \\
        -o conv python tools/prof_conv.py [layer-index ...]
"""
import ctypes as C
import sys

sys.path.insert(0, '.')
import torch

from bench import RESNET_LAYERS
from paper_2301_11659_b200 import _lib

ctx = _lib.Context(0)
L = _lib.lib()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
sel = [int(x) for x in sys.argv[1:]] or list(range(len(RESNET_LAYERS)))
for i in sel:
    name, c, k, r, h = RESNET_LAYERS[i]
    n, oh = 256, h - r + 1
    x = torch.empty(n, c, h, h, device="cuda").uniform_(-1, 1)
    w = torch.empty(k, c, r, r, device="cuda").uniform_(-1, 1)
    y = torch.empty(n, k, oh, oh, device="cuda")

    def run():
        _lib.check(ctx.handle, L.atc_conv2d_nchw_device(ctx.handle, x.data_ptr(), w.data_ptr(), y.data_ptr(), n, c, h,
                                                        h, k, r, r, _lib.PREC_TF32, C.c_void_p(s.cuda_stream)))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    run()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(name, "ok")
