import sys, ctypes as C
sys.path.insert(0, '.')
import torch
from paper_2301_11659_b200 import _lib
ctx = _lib.Context(0)
L = _lib.lib()
m = n = k = 8192
a = torch.rand(m, k, device="cuda") * 2 - 1
b = torch.rand(k, n, device="cuda") * 2 - 1
c = torch.empty(m, n, device="cuda")
s = torch.cuda.current_stream()
for prec in (0, 1):
    for _ in range(2):
        _lib.check(ctx.handle, L.atc_sgemm_rm_device(ctx.handle, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, prec, C.c_void_p(s.cuda_stream)))
torch.cuda.synchronize()
print("ok", float(c[0, 0]))
