"""Extended specs: gemm_ext (transA/transB, alpha/beta,
lda/ldb/ldc) and conv2d_ext (stride, zero padding, dilation).

The reference has no semantics for these (run_dispatch ignores float scalars,
rewriter.cpp:130-132; its conv2d is valid/unit-stride, equivalence.cpp:67-93), so
they are defined in include/atc_b200.h ("Extended semantics"), stated on the CPU
by oracle/ext_oracle.c (pinned by hand-derived known answers) and evaluated on the
GPU by atc_eval_bindings_ext (csrc/eval_ext.cu).

Binding space of an extended spec over a user function: the array permutations of
Appendix C times, per non-array API param in spec order (first param fastest), a
digit whose radix is the number of user ints (plain size params), the size of the
param's constant domain (trans, stride, pad, dil) or the number of user floats
plus the constant domain (alpha, beta).  For a base spec this is exactly the
Appendix C order.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from . import _lib
from .spec import ApiSpec, ext_constants, ext_desc, parse_api_spec

SPECS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "specs")


def spec(name: str) -> ApiSpec:
    """gemm_ext / conv2d_ext (paper_2301_11659_b200/specs/)."""
    with open(os.path.join(SPECS, name + ".json")) as f:
        return parse_api_spec(json.load(f))


class ExtSpace:
    def __init__(self, user_ptrs: list, user_ints: list, user_floats: list, spec: ApiSpec):
        self.spec = spec
        self.user_ptrs, self.user_ints, self.user_floats = list(user_ptrs), list(user_ints), list(user_floats)
        nP, nA = len(self.user_ptrs), len(spec.arrays())
        perms, sel, used = [], [0] * nA, [False] * nP

        def rec(i):
            if i == nA:
                perms.append(list(sel))
                return
            for j in range(nP):
                if not used[j]:
                    used[j] = True
                    sel[i] = j
                    rec(i + 1)
                    used[j] = False

        rec(0)
        self.perms = np.asarray(perms, dtype=np.uint8).reshape(-1, nA)
        self.iconst, self.fconst = ext_constants(spec)
        nI, nF = len(self.user_ints), len(self.user_floats)
        # per non-array param (spec order): ("int", q, choices) / ("float", f, choices);
        # a choice is the ABI map entry (user index, or n_user + constant index)
        self.digits = []
        q = f = 0
        for p in spec.params:
            if p.kind == "int":
                ch = [nI + self.iconst.index(int(v)) for v in p.domain] if p.domain else list(range(nI))
                self.digits.append(("int", q, ch))
                q += 1
            elif p.kind == "float":
                ch = list(range(nF)) + [nF + self.fconst.index(float(v)) for v in p.domain]
                self.digits.append(("float", f, ch))
                f += 1
        self.nS, self.nF = q, f
        self.maps = 1
        for _, _, ch in self.digits:
            self.maps *= len(ch)
        self.count = len(perms) * self.maps

    def decode(self, idx) -> tuple:
        """(arr_map [n, nA], size_map [n, nS], float_map [n, nF]) in the ABI encoding."""
        idx = np.asarray(idx, dtype=np.uint64)
        perm = idx // np.uint64(self.maps)
        s = idx - perm * np.uint64(self.maps)
        am = self.perms[perm.astype(np.int64)]
        sm = np.zeros((len(idx), self.nS), dtype=np.uint8)
        fm = np.zeros((len(idx), max(self.nF, 1)), dtype=np.uint8)
        for kind, i, ch in self.digits:
            r = np.uint64(len(ch))
            d = (s % r).astype(np.int64)
            s = s // r
            (sm if kind == "int" else fm)[:, i] = np.asarray(ch, dtype=np.uint8)[d]
        return am, sm, fm[:, :self.nF]

    def binding(self, idx: int) -> dict:
        am, sm, fm = self.decode([idx])
        nI, nF = len(self.user_ints), len(self.user_floats)
        out = {"arrays": {p.name: self.user_ptrs[am[0, a]] for a, p in enumerate(self.spec.arrays())}}
        sizes, floats = {}, {}
        for q, p in enumerate(self.spec.size_params()):
            e = int(sm[0, q])
            sizes[p.name] = self.user_ints[e] if e < nI else self.iconst[e - nI]
        for f, p in enumerate(self.spec.float_scalars()):
            e = int(fm[0, f])
            floats[p.name] = self.user_floats[e] if e < nF else self.fconst[e - nF]
        out["sizes"], out["floats"] = sizes, floats
        return out


def space_of(program, spec: ApiSpec) -> ExtSpace:
    """The extended space of a fixture program (fixtures.Program)."""
    floats = [p.name for p in program.params if p.kind == "float"]
    return ExtSpace(program.user_ptrs, program.user_ints, floats, spec)


def eval_bindings_ext(ctx: "_lib.Context", spec: ApiSpec, ts, arr_map, size_map, float_map):
    """atc_eval_bindings_ext: (fail_t, reason, first_pass) per binding (FP64, exact)."""
    d = ext_desc(spec)
    h = ts.upload(ctx)
    n = int(arr_map.shape[0])
    am = np.ascontiguousarray(arr_map, dtype=np.uint8)
    sm = np.ascontiguousarray(size_map, dtype=np.uint8)
    fm = np.ascontiguousarray(float_map, dtype=np.uint8) if d.n_floats else np.zeros((n, 1), np.uint8)
    ft = np.empty(n, dtype=np.int8)
    rs = np.empty(n, dtype=np.int8)
    first = C.c_int64(-1)
    _lib.check(ctx.handle, _lib.lib().atc_eval_bindings_ext(ctx.handle, C.byref(d), h.value, am.ctypes.data,
                                                           sm.ctypes.data, fm.ctypes.data, n, ft.ctypes.data,
                                                           rs.ctypes.data, C.byref(first)))
    return ft, rs, int(first.value)


def run_reference_ext(ctx: "_lib.Context", spec: ApiSpec, sizes: list, floats: list, bufs: list, is_f32: list):
    """atc_run_reference_ext on host buffers (rewritten in place); raises AtcError
    (ATC_ERR_DISPATCH) where the dispatch checks fail."""
    d = ext_desc(spec)
    sz = np.ascontiguousarray(sizes, dtype=np.int64)
    fl = np.ascontiguousarray(floats if len(floats) else [0.0], dtype=np.float64)
    ptrs = (C.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
    lens = np.asarray([len(b) for b in bufs], dtype=np.int64)
    f32 = np.asarray(is_f32, dtype=np.int32)
    _lib.check(ctx.handle, _lib.lib().atc_run_reference_ext(ctx.handle, C.byref(d), sz.ctypes.data, fl.ctypes.data,
                                                           C.cast(ptrs, C.c_void_p), lens.ctypes.data,
                                                           f32.ctypes.data))
