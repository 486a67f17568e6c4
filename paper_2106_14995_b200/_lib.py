"""ctypes binding of include/tb_capi.h (libtronbatch_b200.so, built in-tree).

There is no fallback: if the shared library is missing or cannot be loaded
this module raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TB_LIB_PATH") or os.path.join(_HERE, "libtronbatch_b200.so")

TB_OK = 0
TB_E_INVALID_ARGUMENT = 1
TB_E_CUDA = 2
TB_E_NCCL = 3
TB_E_PROBLEM = 4

TB_MEM_HOST = 0
TB_MEM_DEVICE = 1

TB_FAMILY_HS45 = 0
TB_FAMILY_BOXQP = 1
TB_FAMILY_NCVX = 2
TB_FAMILY_BRANCH = 3


class TronConfigC(C.Structure):
    _fields_ = [
        ("tol_pg", C.c_double),
        ("has_delta0", C.c_int32),
        ("delta0", C.c_double),
        ("max_iter", C.c_int32),
        ("cg_tol", C.c_double),
        ("eta0", C.c_double),
        ("sigma1", C.c_double),
        ("sigma2", C.c_double),
        ("sigma3", C.c_double),
        ("mu0", C.c_double),
        ("mu1", C.c_double),
        ("interp_factor", C.c_double),
        ("delta_max", C.c_double),
    ]


class ProblemBatchC(C.Structure):
    _fields_ = [
        ("family", C.c_int32),
        ("dim", C.c_int32),
        ("count", C.c_int64),
        ("x0", C.c_void_p),
        ("lower", C.c_void_p),
        ("upper", C.c_void_p),
        ("params", C.c_void_p),
        ("params_stride", C.c_int64),
        ("memspace", C.c_int32),
    ]


class BatchResultC(C.Structure):
    _fields_ = [
        ("x_star", C.c_void_p),
        ("f_star", C.c_void_p),
        ("pg_norm", C.c_void_p),
        ("status", C.c_void_p),
        ("iterations", C.c_void_p),
        ("cg_iterations", C.c_void_p),
        ("f_evals", C.c_void_p),
        ("wall_time", C.c_void_p),
        ("flops", C.c_void_p),
        ("memspace", C.c_int32),
        ("partition_times", C.c_double * 64),
        ("n_partitions", C.c_int32),
        ("batch_wall_time", C.c_double),
        ("kernel_time", C.c_double),
    ]


# tb_pack_fn / tb_unpack_fn (tb_solve_batch_packed's per-chunk callbacks)
PACK_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
UNPACK_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(BatchResultC))

# every symbol include/tb_capi.h declares, with its ctypes signature
SIGNATURES = {
    "tb_config_default": (None, [C.POINTER(TronConfigC)]),
    "tb_config_validate": (C.c_int, [C.POINTER(TronConfigC)]),
    "tb_family_nparams": (C.c_int64, [C.c_int32, C.c_int32]),
    "tb_context_create": (C.c_int, [C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_void_p)]),
    "tb_context_destroy": (C.c_int, [C.c_void_p]),
    "tb_context_set_mode": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    "tb_context_set_form": (C.c_int, [C.c_void_p, C.c_int32]),
    "tb_context_set_order": (C.c_int, [C.c_void_p, C.c_int32]),
    "tb_solve_batch": (
        C.c_int,
        [C.c_void_p, C.POINTER(ProblemBatchC), C.POINTER(TronConfigC), C.POINTER(BatchResultC)],
    ),
    "tb_solve_batch_async": (
        C.c_int,
        [C.c_void_p, C.POINTER(ProblemBatchC), C.POINTER(TronConfigC), C.POINTER(BatchResultC), C.c_void_p],
    ),
    "tb_solve_batch_packed": (
        C.c_int,
        [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.POINTER(TronConfigC), PACK_FN, UNPACK_FN, C.c_void_p,
         C.POINTER(BatchResultC)],
    ),
    "tb_imbalance": (
        C.c_int,
        [
            C.POINTER(C.c_double),
            C.c_int32,
            C.c_int32,
            C.POINTER(C.c_double),
            C.POINTER(C.c_double),
            C.POINTER(C.c_double),
            C.POINTER(C.c_double),
        ],
    ),
    "tb_last_error": (C.c_char_p, []),
    "tb_kernel_launch_count": (C.c_int64, []),
    "tb_measure_fp64_peak": (C.c_int, [C.c_int32, C.POINTER(C.c_double)]),
    "tb_host_alloc": (C.c_int, [C.c_int64, C.POINTER(C.c_void_p)]),
    "tb_host_free": (C.c_int, [C.c_void_p]),
}

_lib = None


def load() -> C.CDLL:
    """Load the in-tree CUDA library (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("TB_LIB_PATH") and not hasattr(lib, name):
            continue  # A/B experiments against an older library build
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().tb_last_error().decode(errors="replace")
