"""ctypes binding of libatc_b200.so (include/atc_b200.h).

The product path has no fallback: if the library cannot be loaded, or no sm_100
device is present when a compute entry point is called, an AtcError is raised.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libatc_b200.so")

ATC_MAX_ARRAYS = 4
ATC_MAX_SIZES = 12
ATC_MAX_DIMS = 6
ATC_SZ_COUNT = 15

ATC_OK = 0
ATC_ERR_ARG = -1
ATC_ERR_CUDA = -2
ATC_ERR_DEVICE = -3
ATC_ERR_DISPATCH = -4

SEM_GEMM, SEM_CONV2D = 0, 1
LAYOUT_ROW, LAYOUT_COL = 0, 1
# size roles, in ATC_SZ_* order
SIZE_ROLES = ["m", "n", "k", "lda", "ldb", "ldc"]
CONV_SIZE_ROLES = ["n", "c", "h", "w", "k", "r", "s", "oh", "ow"]
ARRAY_ROLES = {"gemm": {"a": 0, "b": 1, "c": 2}, "conv2d": {"in": 0, "weights": 1, "out": 2}}

PASS, FAIL_MISMATCH, FAIL_DISPATCH, FAIL_TESTSET, FAIL_UB = 0, 1, 2, 3, 4
REASON_NAMES = ["pass", "mismatch", "dispatch_failed", "testset", "ub"]
MODE_FP64, MODE_FP32_SCREEN = 0, 1
PREC_TF32, PREC_3XTF32 = 0, 1


class AtcError(RuntimeError):
    """A failing status from libatc_b200 (the message is atc_last_error)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class SpecDesc(C.Structure):
    _fields_ = [
        ("semantics", C.c_int32),
        ("layout", C.c_int32),
        ("n_arrays", C.c_int32),
        ("n_sizes", C.c_int32),
        ("array_role", C.c_int32 * ATC_MAX_ARRAYS),
        ("array_livein", C.c_int32 * ATC_MAX_ARRAYS),
        ("array_ndims", C.c_int32 * ATC_MAX_ARRAYS),
        ("array_dims", (C.c_int32 * ATC_MAX_DIMS) * ATC_MAX_ARRAYS),
        ("role_size", C.c_int32 * ATC_SZ_COUNT),
    ]


class Testsets(C.Structure):
    _fields_ = [
        ("n_tests", C.c_int32),
        ("n_ints", C.c_int32),
        ("n_ptrs", C.c_int32),
        ("int_values", C.POINTER(C.c_int64)),
        ("ptr_is_f32", C.POINTER(C.c_int32)),
        ("region_len", C.POINTER(C.c_int64)),
        ("init", C.POINTER(C.c_void_p)),
        ("final_", C.POINTER(C.c_void_p)),
        ("test_ok", C.POINTER(C.c_int32)),
        ("n_floats", C.c_int32),
        ("float_values", C.c_void_p),
    ]


SEM_GEMM_EXT, SEM_CONV2D_EXT = 2, 3
ATC_XR_COUNT, ATC_FR_COUNT, ATC_MAX_FLOATS, ATC_MAX_CONSTS = 8, 2, 4, 8
EXT_SIZE_ROLES = ["transa", "transb", "stride_h", "stride_w", "pad_h", "pad_w", "dil_h", "dil_w"]
EXT_FLOAT_ROLES = ["alpha", "beta"]


class SpecExt(C.Structure):
    """atc_spec_ext (include/atc_b200.h, "Extended semantics")."""

    _fields_ = [
        ("base", SpecDesc),
        ("n_floats", C.c_int32),
        ("ext_role_size", C.c_int32 * ATC_XR_COUNT),
        ("role_float", C.c_int32 * ATC_FR_COUNT),
        ("n_iconst", C.c_int32),
        ("n_fconst", C.c_int32),
        ("iconst", C.c_int64 * ATC_MAX_CONSTS),
        ("fconst", C.c_double * ATC_MAX_CONSTS),
    ]


class SeededTestsets(C.Structure):
    """atc_seeded_testsets (include/atc_b200.h)."""

    _fields_ = [
        ("n_tests", C.c_int32),
        ("n_ints", C.c_int32),
        ("n_ptrs", C.c_int32),
        ("int_values", C.c_void_p),
        ("ptr_is_f32", C.c_void_p),
        ("region_len", C.c_void_p),
        ("test_ok", C.c_void_p),
        ("stream_seed", C.c_void_p),
        ("stream_skip", C.c_void_p),
        ("diff_off", C.c_void_p),
        ("diff_pos", C.c_void_p),
        ("diff_val", C.c_void_p),
        ("needed_only", C.c_int32),
    ]


class PrefixTestsets(C.Structure):
    """atc_prefix_testsets (include/atc_b200.h)."""

    _fields_ = [
        ("n_tests", C.c_int32),
        ("n_ints", C.c_int32),
        ("n_ptrs", C.c_int32),
        ("int_values", C.c_void_p),
        ("ptr_is_f32", C.c_void_p),
        ("region_len", C.c_void_p),
        ("test_ok", C.c_void_p),
        ("init", C.c_void_p),
        ("diff_off", C.c_void_p),
        ("diff_pos", C.c_void_p),
        ("diff_val", C.c_void_p),
    ]


class Profile(C.Structure):
    _fields_ = [
        ("screen_ms", C.c_double),
        ("screen_launches", C.c_int64),
        ("confirm_ms", C.c_double),
        ("confirm_launches", C.c_int64),
        ("survivors", C.c_int64),
        ("bindings", C.c_int64),
        ("kernels", C.c_int64),
    ]


def out_view(jobs, n: int, fields: list):
    """A numpy structured view of the named integer fields of a ctypes array of job
    structures (read after a run: one vectorised read instead of ~4 us of ctypes
    attribute access per job and field)."""
    E = type(jobs)._type_
    fmt = {C.c_int64: np.int64, C.c_int32: np.int32, C.c_uint64: np.uint64}
    formats = []
    for f in fields:
        t = dict(E._fields_)[f]
        formats.append((np.int64, t._length_) if issubclass(t, C.Array) else fmt[t])
    dt = np.dtype({"names": fields, "formats": formats, "offsets": [getattr(E, f).offset for f in fields],
                   "itemsize": C.sizeof(E)})
    return np.frombuffer(jobs, dtype=dt)[:n]


class EnumJob(C.Structure):
    """atc_enum_job (include/atc_b200.h)."""

    _fields_ = [
        ("spec", C.c_void_p),
        ("ts", C.c_void_p),
        ("perms", C.c_void_p),
        ("n_perms", C.c_int32),
        ("begin", C.c_uint64),
        ("end", C.c_uint64),
        ("survivors", C.c_void_p),
        ("cap", C.c_int64),
        ("n_survivors", C.c_int64),
        ("reason_counts", C.c_int64 * 5),
        ("status", C.c_int32),
    ]


class BindJob(C.Structure):
    """atc_bind_job (include/atc_b200.h)."""

    _fields_ = [
        ("spec", C.c_void_p),
        ("ts", C.c_void_p),
        ("arr_map", C.c_void_p),
        ("size_map", C.c_void_p),
        ("n_bindings", C.c_int64),
        ("fail_t", C.c_void_p),
        ("reason", C.c_void_p),
        ("first_pass", C.c_int64),
        ("status", C.c_int32),
    ]


class GroupJob(C.Structure):
    """atc_group_job (include/atc_b200.h)."""

    _fields_ = [
        ("spec", C.c_void_p),
        ("ts", C.c_void_p),
        ("perms", C.c_void_p),
        ("n_perms", C.c_int32),
        ("begin", C.c_uint64),
        ("end", C.c_uint64),
        ("survivors", C.c_void_p),
        ("cap", C.c_int64),
        ("n_survivors", C.c_int64),
        ("reason_counts", C.c_int64 * 5),
        ("first_pass", C.c_int64),
        ("status", C.c_int32),
    ]


OPT_CONV_SCREEN, OPT_TC_FLAGS, OPT_CONV_STREAMS, OPT_SMALL_LOG2, OPT_K2B_PARTS = 0, 1, 2, 3, 4
CONV_SCREEN_AUTO, CONV_SCREEN_PLANES, CONV_SCREEN_GENERIC = 0, 1, 2
TC_NO_KSPLIT, TC_NO_2SM, TC_NO_TMA_STORE, TC_NO_PAIR, TC_NO_IM2COL, TC_B_KMAJOR, TC_NO_SWAP1X1 = 1, 2, 4, 8, 16, 32, 64
TC_NO_B3D = 128

# (name, restype, argtypes) for every function declared in include/atc_b200.h
_P = C.c_void_p
_SIGS = [
    ("atc_device_count", C.c_int, []),
    ("atc_create", _P, [C.c_int]),
    ("atc_destroy", None, [_P]),
    ("atc_last_error", C.c_char_p, [_P]),
    ("atc_set_option", C.c_int, [_P, C.c_int32, C.c_int32]),
    ("atc_set_stream", C.c_int, [_P, _P]),
    ("atc_profile_start", C.c_int, [_P]),
    ("atc_profile_read", C.c_int, [_P, C.POINTER(Profile)]),
    ("atc_measure_dfma_peak", C.c_int, [_P, C.POINTER(C.c_double)]),
    ("atc_testsets_upload", C.c_int, [_P, C.POINTER(Testsets), C.POINTER(_P)]),
    ("atc_testsets_free", C.c_int, [_P, _P]),
    ("atc_testsets_upload_async", C.c_int, [_P, C.POINTER(Testsets), C.POINTER(_P)]),
    ("atc_testsets_upload_seeded", C.c_int, [_P, C.POINTER(SeededTestsets), C.POINTER(_P)]),
    ("atc_testsets_upload_prefix", C.c_int, [_P, C.POINTER(PrefixTestsets), C.POINTER(_P)]),
    ("atc_testsets_update_seeded", C.c_int, [_P, _P, C.POINTER(SeededTestsets)]),
    ("atc_testsets_update_seeded_many", C.c_int, [_P, _P, C.POINTER(SeededTestsets), C.c_int32]),
    ("atc_testsets_download", C.c_int, [_P, _P, _P, _P]),
    ("atc_eval_bindings", C.c_int, [_P, C.POINTER(SpecDesc), _P, _P, _P, C.c_int64, C.c_int32, _P, _P,
                                    C.POINTER(C.c_int64)]),
    ("atc_eval_bindings_many", C.c_int, [_P, C.POINTER(BindJob), C.c_int32, C.c_int32]),
    ("atc_eval_bindings_device", C.c_int, [_P, C.POINTER(SpecDesc), _P, _P, _P, C.c_int64, C.c_int32, _P, _P, _P]),
    ("atc_eval_enumerated", C.c_int, [_P, C.POINTER(SpecDesc), _P, _P, C.c_int32, C.c_uint64, C.c_uint64, C.c_int32,
                                      _P, C.c_int64, C.POINTER(C.c_int64), _P]),
    ("atc_eval_enumerated_many", C.c_int, [_P, C.POINTER(EnumJob), C.c_int32, C.c_int32]),
    ("atc_enum_batch_create", _P, [_P, C.POINTER(EnumJob), C.c_int32, C.c_int32]),
    ("atc_enum_batch_run", C.c_int, [_P, _P]),
    ("atc_enum_batch_destroy", None, [_P, _P]),
    ("atc_group_create", _P, [_P, C.c_int32]),
    ("atc_group_destroy", None, [_P]),
    ("atc_group_last_error", C.c_char_p, [_P]),
    ("atc_group_size", C.c_int32, [_P]),
    ("atc_group_member", _P, [_P, C.c_int32]),
    ("atc_group_testsets_upload_seeded", C.c_int, [_P, C.POINTER(SeededTestsets), C.POINTER(_P)]),
    ("atc_group_testsets_upload_prefix", C.c_int, [_P, C.POINTER(PrefixTestsets), C.POINTER(_P)]),
    ("atc_group_testsets_free", C.c_int, [_P, _P]),
    ("atc_group_testsets_member", _P, [_P, C.c_int32]),
    ("atc_group_eval_enumerated_many", C.c_int, [_P, C.POINTER(GroupJob), C.c_int32, C.c_int32]),
    ("atc_group_batch_create", _P, [_P, C.POINTER(GroupJob), C.c_int32, C.c_int32]),
    ("atc_group_batch_run", C.c_int, [_P, _P]),
    ("atc_group_batch_destroy", None, [_P, _P]),
    ("atc_plan_shards", C.c_int, [_P, C.c_int32, C.c_int32, _P, _P]),
    ("atc_eval_bindings_ext", C.c_int, [_P, C.POINTER(SpecExt), _P, _P, _P, _P, C.c_int64, _P, _P,
                                        C.POINTER(C.c_int64)]),
    ("atc_run_reference_ext", C.c_int, [_P, C.POINTER(SpecExt), _P, _P, _P, _P, _P]),
    ("atc_run_reference", C.c_int, [_P, C.POINTER(SpecDesc), _P, _P, _P]),
    ("atc_dispatch", C.c_int, [_P, C.POINTER(SpecDesc), _P, _P, _P, _P]),
    ("atc_sgemm_rm", C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int64, C.c_int64, C.c_int32]),
    ("atc_sgemm_rm_device", C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int64, C.c_int64, C.c_int32, _P]),
    ("atc_conv2d_nchw", C.c_int, [_P, _P, _P, _P] + [C.c_int64] * 7 + [C.c_int32]),
    ("atc_conv2d_nchw_device", C.c_int, [_P, _P, _P, _P] + [C.c_int64] * 7 + [C.c_int32, _P]),
    ("atc_mt64_raw", None, [C.c_uint64, C.c_uint64, C.c_int64, _P]),
    ("atc_mt64_uniform", None, [C.c_uint64, C.c_uint64, C.c_int64, C.c_double, C.c_double, C.c_int32, _P]),
]
EXPORTED = [s[0] for s in _SIGS]

_lib = None


def lib():
    """Load libatc_b200.so once; raise loudly if it is missing or incomplete."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise AtcError(ATC_ERR_DEVICE, f"{LIB_PATH} is not built (run __graft_entry__.build())")
    h = C.CDLL(LIB_PATH)
    for name, res, args in _SIGS:
        fn = getattr(h, name)  # AttributeError if the symbol is missing
        fn.restype = res
        fn.argtypes = args
    _lib = h
    return h


def check(ctx, rc: int) -> None:
    if rc != ATC_OK:
        msg = lib().atc_last_error(ctx)
        raise AtcError(rc, msg.decode() if msg else f"atc error {rc}")


class Context:
    """One libatc context bound to one CUDA device (one process per GPU)."""

    def __init__(self, device: int = 0):
        L = lib()
        self.device = device
        self.handle = L.atc_create(device)
        if not self.handle:
            raise AtcError(ATC_ERR_DEVICE, "atc_create returned NULL")
        msg = L.atc_last_error(self.handle)
        if msg:
            err = msg.decode()
            L.atc_destroy(self.handle)
            self.handle = None
            raise AtcError(ATC_ERR_DEVICE, err)

    def set_option(self, option: int, value: int) -> None:
        """atc_set_option: kernel-variant selection (A/B checks)."""
        check(self.handle, lib().atc_set_option(self.handle, option, value))

    def close(self) -> None:
        if self.handle:
            lib().atc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default = {}


def default_context(device: int = 0) -> Context:
    ctx = _default.get(device)
    if ctx is None:
        ctx = _default[device] = Context(device)
    return ctx
