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
