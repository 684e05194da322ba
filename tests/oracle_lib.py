"""ctypes access to the CPU oracle (oracle/liboracle_p2.so) — test-only checker."""
import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle")
SO = os.path.join(ORACLE, "liboracle_p2.so")


class OracleSpec(C.Structure):
    _fields_ = [
        ("semantics", C.c_int32),
        ("layout", C.c_int32),
        ("n_arrays", C.c_int32),
        ("n_sizes", C.c_int32),
        ("array_role", C.c_int32 * 4),
        ("array_livein", C.c_int32 * 4),
        ("array_ndims", C.c_int32 * 4),
        ("array_dims", (C.c_int32 * 6) * 4),
        ("role_size", C.c_int32 * 15),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            subprocess.run(["make", "-C", ORACLE, "port"], check=True, capture_output=True)
        _lib = C.CDLL(SO)
        _lib.oracle_fnv1a.restype = C.c_uint64
        _lib.oracle_fnv1a.argtypes = [C.c_void_p, C.c_int64]
        _lib.oracle_run_reference.restype = C.c_int
        _lib.oracle_verify_many.restype = None
        _lib.oracle_cpu_gemm.restype = None
        _lib.oracle_xpu_gemm.restype = None
    return _lib


def spec_struct(spec) -> OracleSpec:
    """Same field meaning as atc_spec_desc; built from the package's decode table."""
    d = spec.to_desc()
    s = OracleSpec()
    C.memmove(C.byref(s), C.byref(d), C.sizeof(OracleSpec))
    return s


def fnv1a(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a)
    return int(lib().oracle_fnv1a(a.ctypes.data, a.nbytes))


def run_reference(spec, sizes: list, bufs: list) -> int:
    s = spec_struct(spec)
    sz = np.asarray(sizes, dtype=np.int64)
    arrs = [np.ascontiguousarray(b, dtype=np.float64) for b in bufs]
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    lens = np.array([len(a) for a in arrs], dtype=np.int64)
    rc = lib().oracle_run_reference(C.byref(s), C.c_void_p(sz.ctypes.data), ptrs, C.c_void_p(lens.ctypes.data))
    for b, a in zip(bufs, arrs):
        if b is not a:
            b[:] = a
    return rc


def verify_many(spec, ts, arr_map: np.ndarray, size_map: np.ndarray, threads: int = 0):
    """Literal verify_rewrite restatement over recorded test sets (RecordedTestsets)."""
    s = spec_struct(spec)
    cs, keep = ts.c_struct()
    n = int(arr_map.shape[0])
    am = np.ascontiguousarray(arr_map, dtype=np.uint8)
    sm = np.ascontiguousarray(size_map, dtype=np.uint8)
    ft = np.empty(n, dtype=np.int8)
    rs = np.empty(n, dtype=np.int8)
    threads = threads or os.cpu_count() or 1
    lib().oracle_verify_many(C.byref(s), cs.n_tests, cs.n_ints, cs.n_ptrs, cs.int_values, cs.ptr_is_f32,
                             cs.region_len, cs.init, cs.final_, cs.test_ok, C.c_void_p(am.ctypes.data),
                             C.c_void_p(sm.ctypes.data), C.c_int64(n), C.c_int(threads),
                             C.c_void_p(ft.ctypes.data), C.c_void_p(rs.ctypes.data))
    del keep
    return ft, rs


def cpu_gemm(a, b, m, n, k):
    c = np.empty(m * n, dtype=np.float32)
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    lib().oracle_cpu_gemm(C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data), C.c_void_p(c.ctypes.data),
                          C.c_int64(m), C.c_int64(n), C.c_int64(k))
    return c.reshape(m, n)


def xpu_gemm(a, b, m, n, k, threads=0):
    c = np.empty(m * n, dtype=np.float32)
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    lib().oracle_xpu_gemm(C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data), C.c_void_p(c.ctypes.data),
                          C.c_int64(m), C.c_int64(n), C.c_int64(k), C.c_int(threads or os.cpu_count() or 1))
    return c.reshape(m, n)


class OracleSpecExt(C.Structure):
    """oracle_spec_ext (oracle/p2_oracle.h): the layout of atc_spec_ext."""

    _fields_ = [
        ("base", OracleSpec),
        ("n_floats", C.c_int32),
        ("ext_role_size", C.c_int32 * 8),
        ("role_float", C.c_int32 * 2),
        ("n_iconst", C.c_int32),
        ("n_fconst", C.c_int32),
        ("iconst", C.c_int64 * 8),
        ("fconst", C.c_double * 8),
    ]


def ext_spec_struct(spec) -> OracleSpecExt:
    from paper_2301_11659_b200.spec import ext_desc

    d = ext_desc(spec)
    s = OracleSpecExt()
    assert C.sizeof(OracleSpecExt) == C.sizeof(d)
    C.memmove(C.byref(s), C.byref(d), C.sizeof(OracleSpecExt))
    return s


def run_ext(spec, sizes: list, floats: list, bufs: list, is_f32: list):
    """oracle_run_ext: (status, detail); bufs (float64 arrays) rewritten in place."""
    s = ext_spec_struct(spec)
    sz = np.ascontiguousarray(sizes, dtype=np.int64)
    fl = np.ascontiguousarray(floats if len(floats) else [0.0], dtype=np.float64)
    ptrs = (C.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
    lens = np.asarray([len(b) for b in bufs], dtype=np.int64)
    f32 = np.asarray(is_f32, dtype=np.int32)
    detail = C.create_string_buffer(128)
    lib().oracle_run_ext.restype = C.c_int
    rc = lib().oracle_run_ext(C.byref(s), C.c_void_p(sz.ctypes.data), C.c_void_p(fl.ctypes.data), ptrs,
                              C.c_void_p(lens.ctypes.data), C.c_void_p(f32.ctypes.data), detail)
    return rc, detail.value.decode()


def verify_ext_many(spec, ts, arr_map, size_map, float_map, threads: int = 0):
    """The extended P2 predicate on the CPU (oracle_verify_ext_many)."""
    s = ext_spec_struct(spec)
    cs, keep = ts.c_struct()
    n = int(arr_map.shape[0])
    am = np.ascontiguousarray(arr_map, dtype=np.uint8)
    sm = np.ascontiguousarray(size_map, dtype=np.uint8)
    fm = np.ascontiguousarray(float_map if float_map.size else np.zeros((n, 1)), dtype=np.uint8)
    fl = np.ascontiguousarray(ts.floats if ts.floats is not None and ts.floats.size else np.zeros((ts.n_tests, 1)),
                              dtype=np.float64)
    nF = 0 if ts.floats is None else ts.floats.shape[1]
    ft = np.empty(n, dtype=np.int8)
    rs = np.empty(n, dtype=np.int8)
    threads = threads or os.cpu_count() or 1
    lib().oracle_verify_ext_many.restype = None
    lib().oracle_verify_ext_many(C.byref(s), cs.n_tests, cs.n_ints, cs.n_ptrs, nF, cs.int_values,
                                 C.c_void_p(fl.ctypes.data), cs.ptr_is_f32, cs.region_len, cs.init, cs.final_,
                                 cs.test_ok, C.c_void_p(am.ctypes.data), C.c_void_p(sm.ctypes.data),
                                 C.c_void_p(fm.ctypes.data), C.c_int64(n), C.c_int(threads),
                                 C.c_void_p(ft.ctypes.data), C.c_void_p(rs.ctypes.data))
    del keep
    return ft, rs
