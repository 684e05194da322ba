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
  make_routed_dispatch         rewriter::make_routed_dispatch (rewriter.cpp:183-213): cpu/xpu
                               labels from the predictor; "xpu" f32 calls -> atc_sgemm_rm /
                               atc_conv2d_nchw, all else exact FP64
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


def _decode(spec: ApiSpec, name: str, args: list, regions: dict):
    """rewriter.cpp:101-134: name, arity and kinds, positional decode."""
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
    return sizes, region_of


def _check_extents(spec: ApiSpec, sizes: dict, region_of: dict, regions: dict) -> None:
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


def _exact(spec: ApiSpec, desc, cx, sizes: dict, region_of: dict, regions: dict) -> None:
    """run_dispatch's compute + write-back (rewriter.cpp:150-161), FP64 on the GPU."""
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


def make_gpu_dispatch(spec: ApiSpec, ctx=None):
    """A DispatchContext handler computing on the GPU (FP64, bit-exact with the
    oracle dispatch).  handler(name, args, regions) mutates regions in place and
    raises RuntimeError exactly where run_dispatch throws."""
    cx = _ctx(ctx)
    desc = spec.to_desc()

    def handler(name: str, args: list, regions: dict) -> None:
        sizes, region_of = _decode(spec, name, args, regions)
        _check_extents(spec, sizes, region_of, regions)
        _exact(spec, desc, cx, sizes, region_of, regions)

    return handler


def _role_size(spec: ApiSpec, sizes: dict, role: str, default: int = 1) -> int:
    """rewriter.cpp:164-172."""
    for p in spec.params:
        if p.kind == "int" and p.role == role and p.name in sizes:
            return sizes[p.name]
    return default


def routed_sizes(spec: ApiSpec, sizes: dict) -> list:
    """The predictor features of one call (rewriter.cpp:194-205): conv as its im2col
    GEMM (filters x batch*out positions, depth c*r*s), gemm as (m, n, k)."""
    r = lambda role: _role_size(spec, sizes, role)  # noqa: E731
    if spec.semantics == "conv2d":
        return [r("k"), r("n") * r("oh") * r("ow"), r("c") * r("r") * r("s")]
    return [r("m"), r("n"), r("k")]


def svm_decision(model: dict, mnk) -> float:
    """profitability::decision_value (profitability.cpp:147-161,281-283) for a model in
    save_svm's JSON form (profitability.cpp:296-311): poly kernel over min-max
    normalised features.  Evaluation only — training stays in the reference (SURVEY
    §8: the SVM is a host model)."""
    k = model.get("kernel", {})
    gamma, coef0, degree = k.get("gamma", 1.0), k.get("coef0", 0.0), k.get("degree", 3)
    lo, hi = model["feat_min"], model["feat_max"]
    x = [((float(mnk[i]) - lo[i]) / (hi[i] - lo[i])) if hi[i] - lo[i] > 0 else 0.5 for i in range(len(lo))]
    v = model.get("b", 0.0)
    for sv, ay in zip(model.get("support", []), model.get("alpha_y", [])):
        dot = 0.0
        for p, q in zip(sv, x):
            dot += p * q
        v += ay * (gamma * dot + coef0) ** degree
    return v


def svm_predictor(model: dict):
    """profitability::predict_backend (profitability.cpp:285-287) bound to one model:
    mnk -> 1 ("xpu") iff the decision value is >= 0, else 0 ("cpu")."""
    return lambda mnk: 1 if svm_decision(model, mnk) >= 0.0 else 0


def _tensor(spec: ApiSpec, cx, prec: int, sizes: dict, region_of: dict, regions: dict) -> bool:
    """The "xpu" leg (integration/atc_liftc_adapter.cpp tensor_dispatch): the call on
    atc_sgemm_rm / atc_conv2d_nchw when every region is f32 and the backends express
    it; False sends the call down the exact path."""
    regs = {p.role: regions[region_of[p.name]] for p in spec.arrays()}
    if any(r.elem != "f32" for r in regs.values()):
        return False
    rs = lambda role, d=0: _role_size(spec, sizes, role, d)  # noqa: E731
    L = _lib.lib()
    if spec.semantics == "gemm":
        m, n, k = rs("m"), rs("n"), rs("k")
        row = spec.layout == "rowmajor"
        lda, ldb, ldc = rs("lda", k if row else m), rs("ldb", n if row else k), rs("ldc", n if row else m)
        if min(m, n, k) < 1 or lda < (k if row else m) or ldb < (n if row else k) or ldc < (n if row else m):
            return False
        A, B, Cr = regs["a"].data, regs["b"].data, regs["c"].data
        i, p, j = np.arange(m)[:, None], np.arange(k)[None, :], np.arange(n)[None, :]
        ia = i * lda + p if row else p * lda + i
        ib = np.arange(k)[:, None] * ldb + j if row else j * ldb + np.arange(k)[:, None]
        ic = i * ldc + j if row else j * ldc + i
        if ia.max() >= len(A) or ib.max() >= len(B) or ic.max() >= len(Cr):
            return False
        a = np.ascontiguousarray(A[ia], dtype=np.float32)
        b = np.ascontiguousarray(B[ib], dtype=np.float32)
        c = np.empty((m, n), dtype=np.float32)
        _lib.check(cx.handle, L.atc_sgemm_rm(cx.handle, a.ctypes.data, b.ctypes.data, c.ctypes.data, m, n, k, prec))
        out = Cr.copy()
        out[ic] = c
        regs["c"].data = out
        return True
    n, c, h, w, k, r, s = (rs(x) for x in ("n", "c", "h", "w", "k", "r", "s"))
    oh, ow = rs("oh", h - r + 1), rs("ow", w - s + 1)
    if min(n, c, k, r, s) < 1 or oh != h - r + 1 or ow != w - s + 1 or oh < 1 or ow < 1 or c % 32:
        return False
    nin, nw, nout = n * c * h * w, k * c * r * s, n * k * oh * ow
    if len(regs["in"].data) < nin or len(regs["weights"].data) < nw or len(regs["out"].data) < nout:
        return False
    x = np.ascontiguousarray(regs["in"].data[:nin], dtype=np.float32)
    wt = np.ascontiguousarray(regs["weights"].data[:nw], dtype=np.float32)
    o = np.empty(nout, dtype=np.float32)
    _lib.check(cx.handle, L.atc_conv2d_nchw(cx.handle, x.ctypes.data, wt.ctypes.data, o.ctypes.data, n, c, h, w, k,
                                            r, s, prec))
    out = regs["out"].data.copy()
    out[:nout] = o
    regs["out"].data = out
    return True


def make_routed_dispatch(spec: ApiSpec, predict=None, choices: list | None = None, precision: str = "exact",
                         ctx=None):
    """rewriter::make_routed_dispatch (rewriter.hpp:57-66, rewriter.cpp:183-213) on the
    GPU.  predict(mnk) -> 0/1 is the backend predictor (svm_predictor(model json) for
    the reference's saved model); each call appends "xpu"/"cpu" to `choices` ("cpu"
    for every call without a predictor).  "xpu" calls on f32 regions run on the
    tcgen05 backends only when the caller opts in with precision "tf32" / "3xtf32";
    by default (precision == "exact") every call — like everything else — runs the
    exact FP64 path, bit-identical to the reference's routed dispatch, which only
    records the label."""
    desc = spec.to_desc()
    if precision != "exact" and precision not in _PREC:
        raise ValueError(f"precision must be 'exact', 'tf32' or '3xtf32', not {precision!r}")

    def handler(name: str, args: list, regions: dict) -> None:
        # the label comes first (rewriter.cpp:190-209), from an arity-clipped decode of
        # the size slots, so a call run_dispatch then rejects is still labelled
        xpu = False
        if predict is not None and choices is not None:
            label_sizes = {ap.name: a.i for ap, a in zip(spec.params, args) if ap.kind == "int"}
            xpu = predict(routed_sizes(spec, label_sizes)) == 1
            choices.append("xpu" if xpu else "cpu")
        elif choices is not None:
            choices.append("cpu")
        sizes, region_of = _decode(spec, name, args, regions)
        cx = _ctx(ctx)  # resolved per call: labels and decode errors need no device
        _check_extents(spec, sizes, region_of, regions)
        if xpu and precision != "exact" and _tensor(spec, cx, _PREC[precision], sizes, region_of, regions):
            return
        _exact(spec, desc, cx, sizes, region_of, regions)

    return handler
