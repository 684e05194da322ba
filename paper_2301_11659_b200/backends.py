"""Replaced-call API backends (host-side mirror of the reference's backend surface).

  sgemm / xpu_gemm / cpu_gemm  profitability::cpu_gemm / xpu_gemm
                               (/root/reference/proj/include/liftc/profitability.hpp:27-28)
                               -> atc_sgemm_rm, tcgen05 kind::tf32 (TF32 or 3xTF32)
  conv2d_nchw                  reference_conv2d semantics on FP32 data -> atc_conv2d_nchw
  run_reference                equivalence::run_reference (equivalence.hpp:53-54), FP64
                               exact on the GPU -> atc_run_reference
  make_gpu_dispatch            rewriter::make_oracle_dispatch (rewriter.hpp:57-66): the
                               DispatchContext handler, same positional decode, checks,
                               error messages ("dispatch arity", "... elements ...") and
                               f32 write-back rounding as run_dispatch (rewriter.cpp:99-162)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .spec import ApiSpec

_PREC = {"tf32": _lib.PREC_TF32, "3xtf32": _lib.PREC_3XTF32}


def _ctx(ctx):
    return ctx or _lib.default_context()


def sgemm(a: np.ndarray, b: np.ndarray, precision: str = "3xtf32", ctx=None) -> np.ndarray:
    """Row-major FP32 C = A @ B on tcgen05 tensor cores (host buffers)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ValueError("inner dimensions differ")
    c = np.empty((m, n), dtype=np.float32)
    cx = _ctx(ctx)
    _lib.check(cx.handle, _lib.lib().atc_sgemm_rm(cx.handle, a.ctypes.data, b.ctypes.data, c.ctypes.data, m, n, k,
                                                  _PREC[precision]))
    return c


def xpu_gemm(a, b, c, m: int, n: int, k: int, precision: str = "3xtf32", ctx=None) -> None:
    """profitability::xpu_gemm signature: flat row-major buffers, C overwritten."""
    out = sgemm(np.asarray(a, dtype=np.float32).reshape(m, k), np.asarray(b, dtype=np.float32).reshape(k, n),
                precision, ctx)
    np.asarray(c).reshape(m, n)[...] = out


cpu_gemm = xpu_gemm  # same contract (profitability.cpp:14-21); both land on the GPU backend


def sgemm_device(a_ptr: int, b_ptr: int, c_ptr: int, m: int, n: int, k: int, precision: str = "tf32",
                 stream: int = 0, ctx=None) -> None:
    """Device-pointer variant on a caller stream (no synchronisation)."""
    cx = _ctx(ctx)
    _lib.check(cx.handle, _lib.lib().atc_sgemm_rm_device(cx.handle, a_ptr, b_ptr, c_ptr, m, n, k, _PREC[precision],
                                                         stream or None))


def conv2d_nchw(x: np.ndarray, w: np.ndarray, precision: str = "3xtf32", ctx=None) -> np.ndarray:
    """out[b,q,y,x] = sum_{z,u,v} in[b,z,y+u,x+v] * w[q,z,u,v] (valid, unit stride)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    n, c, h, ww = x.shape
    k, c2, r, s = w.shape
    if c != c2:
        raise ValueError("channel counts differ")
    out = np.empty((n, k, h - r + 1, ww - s + 1), dtype=np.float32)
    cx = _ctx(ctx)
    _lib.check(cx.handle, _lib.lib().atc_conv2d_nchw(cx.handle, x.ctypes.data, w.ctypes.data, out.ctypes.data, n, c,
                                                     h, ww, k, r, s, _PREC[precision]))
    return out


def conv2d_nchw_device(x_ptr, w_ptr, out_ptr, n, c, h, w, k, r, s, precision="tf32", stream=0, ctx=None) -> None:
    cx = _ctx(ctx)
    _lib.check(cx.handle, _lib.lib().atc_conv2d_nchw_device(cx.handle, x_ptr, w_ptr, out_ptr, n, c, h, w, k, r, s,
                                                            _PREC[precision], stream or None))


def run_reference(spec: ApiSpec, sizes: dict, buffers: dict, ctx=None) -> None:
    """equivalence::run_reference: sizes/buffers keyed by API name; outputs in place."""
    cx = _ctx(ctx)
    desc = spec.to_desc()
    sz = np.array([sizes[p.name] for p in spec.size_params()], dtype=np.int64)
    arrs = [np.ascontiguousarray(buffers[p.name], dtype=np.float64) for p in spec.arrays()]
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    lens = np.array([len(a) for a in arrs], dtype=np.int64)
    _lib.check(cx.handle, _lib.lib().atc_run_reference(cx.handle, C.byref(desc), sz.ctypes.data, ptrs,
                                                       lens.ctypes.data))
    for p, a in zip(spec.arrays(), arrs):
        if isinstance(buffers[p.name], np.ndarray) and buffers[p.name] is not a:
            buffers[p.name][...] = a
        else:
            buffers[p.name] = a


class DispatchArg:
    """interp::DispatchArg (interp.hpp:47-53)."""

    def __init__(self, kind: str, region: str = "", i: int = 0, f: float = 0.0):
        self.kind, self.region, self.i, self.f = kind, region, i, f


class Region:
    def __init__(self, data: np.ndarray, elem: str = "f64"):
        self.data, self.elem = np.ascontiguousarray(data, dtype=np.float64), elem


def make_gpu_dispatch(spec: ApiSpec, ctx=None):
    """A DispatchContext handler computing on the GPU (FP64, bit-exact with the
    oracle dispatch).  handler(name, args, regions) mutates regions in place and
    raises RuntimeError exactly where run_dispatch throws."""
    cx = _ctx(ctx)
    desc = spec.to_desc()

    def handler(name: str, args: list, regions: dict) -> None:
        if name != "atc_dispatch_" + spec.semantics:
            raise RuntimeError(f"dispatch name '{name}' does not match api semantics '{spec.semantics}'")
        if len(args) != len(spec.params):
            raise RuntimeError(f"dispatch arity {len(args)}, api expects {len(spec.params)}")
        sizes, region_of = {}, {}
        for ap, a in zip(spec.params, args):
            if ap.kind == "array":
                if a.kind != "ptr":
                    raise RuntimeError(f"dispatch arg for array '{ap.name}' is not a pointer")
                if a.region not in regions:
                    raise RuntimeError(f"dispatch region '{a.region}' missing")
                region_of[ap.name] = a.region
            elif ap.kind == "int":
                if a.kind != "int":
                    raise RuntimeError(f"dispatch arg for size '{ap.name}' is not an int")
                sizes[ap.name] = a.i
        for ap in spec.arrays():  # rewriter.cpp:136-148
            extent = 1
            for d in ap.dims:
                v = sizes.get(d, -1)
                if v < 1:
                    raise RuntimeError(f"dispatch size '{d}' is not positive")
                extent *= v
            have = len(regions[region_of[ap.name]].data)
            if have < extent:
                raise RuntimeError(f"region bound to '{ap.name}' holds {have} elements, call needs {extent}")
        sz = np.array([sizes[p.name] for p in spec.size_params()], dtype=np.int64)
        arrays = spec.arrays()
        # full-region copies (rewriter.cpp:121); outputs written back below
        bufs = [regions[region_of[p.name]].data.copy() for p in arrays]
        ptrs = (C.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
        lens = np.array([len(b) for b in bufs], dtype=np.int64)
        f32 = np.array([1 if regions[region_of[p.name]].elem == "f32" else 0 for p in arrays], dtype=np.int32)
        _lib.check(cx.handle, _lib.lib().atc_dispatch(cx.handle, C.byref(desc), sz.ctypes.data, ptrs,
                                                      lens.ctypes.data, f32.ctypes.data))
        for p, b in zip(arrays, bufs):
            if p.liveness != "livein":
                regions[region_of[p.name]].data = b

    return handler
