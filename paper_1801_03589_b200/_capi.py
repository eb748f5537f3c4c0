"""ctypes binding of libnesa_b200.so (include/nesa_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  Loading fails loudly if it is missing: there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NESA_LIB") or os.path.join(_HERE, "libnesa_b200.so")  # NESA_LIB: A/B builds

NESA_ABI_VERSION = 3
NESA_PLAN_FAR_ONLY = 1
NESA_PLAN_OCTREE = 2
NESA_PLAN_COMPLEX_NEAR = 4
NESA_PLAN_STORED_VU = 8
NESA_PLAN_HELMHOLTZ_NEAR = 16
NESA_OK = 0
NESA_ERR_INVALID = 1
NESA_ERR_CUDA = 2
NESA_ERR_OOM = 3
NESA_ERR_UNSUPPORTED = 4
NESA_F64 = 0
NESA_F32 = 1
NESA_NEAR = 1
NESA_FAR = 2
NESA_PROFILE = 16
NESA_PROFILE_NEAR = 32

STAT = {"near_entries": 0, "v_entries": 1, "u_entries": 2, "d_refs": 3, "n_dtab": 4,
        "device_bytes": 5, "near_ctas": 6, "kernels_per_matvec": 7, "v_moments": 8,
        "u_terms": 9, "graph_captures": 10, "graphs_cached": 11, "near_wide": 12,
        "far_wide": 13}
STAGE = {"total": 0, "near": 1, "far": 2, "reception": 3}

EXPORTED_SYMBOLS = (
    "nesa_plan_create", "nesa_matvec", "nesa_matvec_stage", "nesa_plan_s_dev",
    "nesa_plan_destroy", "nesa_last_error", "nesa_abi_version", "nesa_plan_stat",
    "nesa_profile_reset", "nesa_profile_read", "nesa_trace_read", "nesa_trace_name",
    "nesa_ktrace_enable", "nesa_ktrace_read", "nesa_dense_matvec", "nesa_matvec_cols",
    "nesa_tree_build", "nesa_tree_error", "nesa_tree_size", "nesa_tree_copy", "nesa_tree_free",
    "nesa_exchange_pack", "nesa_exchange_combine", "nesa_plan_create_dist", "nesa_nccl_unique_id",
    "nesa_nccl_comm_init", "nesa_nccl_comm_destroy", "nesa_matvec_near_wide",
    "nesa_gs_work_bytes", "nesa_gs_step", "nesa_gs_step_shifted", "nesa_gs_last_error",
)

_p = ctypes.c_void_p
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class NesaPlanDesc(ctypes.Structure):
    """Mirror of ``struct nesa_plan_desc`` (field order matters)."""

    _fields_ = [
        ("abi_version", ctypes.c_int32), ("op_dtype", ctypes.c_int32),
        ("Q", ctypes.c_int32), ("n_check", ctypes.c_int32),
        ("N", ctypes.c_int64), ("n_leaves", ctypes.c_int64), ("n_groups", ctypes.c_int64),
        ("l0", ctypes.c_int32), ("L", ctypes.c_int32),
        ("perm", _i64p), ("group_start", _i64p), ("group_stop", _i64p),
        ("parent", _i64p), ("quad", _i32p), ("level_first", _i64p),
        ("level_count", _i64p), ("nbr_ptr", _i64p), ("nbr_idx", _i64p),
        ("int_ptr", _i64p), ("int_idx", _i64p), ("int_dtab", _i64p),
        ("C", _f64p), ("B", _f64p), ("D", _f64p), ("n_dtab", ctypes.c_int64),
        ("near_blob", _f64p), ("V_blob", _f64p), ("U_blob", _f64p),
        ("points_tree", _f64p), ("leaf_center", _f64p), ("leaf_r_check", _f64p),
        ("leaf_r_inaux", _f64p), ("out_fit_leaf", _f64p),
        ("check_cos", _f64p), ("check_sin", _f64p), ("aux_cos", _f64p), ("aux_sin", _f64p),
        ("leaf_begin", ctypes.c_int64), ("leaf_end", ctypes.c_int64),
        ("options", ctypes.c_uint32),
        ("points3", _f64p), ("wavenumber", ctypes.c_double),
    ]


class NesaExchangeDesc(ctypes.Structure):
    """Mirror of ``struct nesa_exchange_desc``."""

    _fields_ = [
        ("n_export", ctypes.c_int64), ("export_ids", _i64p), ("max_export", ctypes.c_int64),
        ("n_import", ctypes.c_int64), ("import_ids", _i64p), ("max_contrib", ctypes.c_int32),
        ("contrib", _i64p),
    ]


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the NESA matvec has no CPU fallback)")
    lib = ctypes.CDLL(path)
    lib.nesa_plan_create.argtypes = [ctypes.POINTER(NesaPlanDesc), ctypes.c_int,
                                     ctypes.POINTER(_p)]
    lib.nesa_plan_create.restype = ctypes.c_int
    lib.nesa_matvec.argtypes = [_p, _p, _p, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, _p]
    lib.nesa_matvec.restype = ctypes.c_int
    lib.nesa_matvec_stage.argtypes = [_p, ctypes.c_int32, _p, _p, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_uint32, _p]
    lib.nesa_matvec_stage.restype = ctypes.c_int
    lib.nesa_plan_s_dev.argtypes = [_p, ctypes.c_int32]
    lib.nesa_plan_s_dev.restype = _p
    lib.nesa_plan_destroy.argtypes = [_p]
    lib.nesa_plan_destroy.restype = ctypes.c_int
    lib.nesa_last_error.argtypes = []
    lib.nesa_last_error.restype = ctypes.c_char_p
    lib.nesa_abi_version.argtypes = []
    lib.nesa_abi_version.restype = ctypes.c_int
    lib.nesa_plan_stat.argtypes = [_p, ctypes.c_int32]
    lib.nesa_plan_stat.restype = ctypes.c_int64
    lib.nesa_profile_reset.argtypes = [_p]
    lib.nesa_profile_reset.restype = ctypes.c_int
    lib.nesa_profile_read.argtypes = [_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_float),
                                      ctypes.c_int32]
    lib.nesa_profile_read.restype = ctypes.c_int
    lib.nesa_trace_read.argtypes = [_p, ctypes.POINTER(ctypes.c_float), ctypes.c_int32]
    lib.nesa_trace_read.restype = ctypes.c_int
    lib.nesa_trace_name.argtypes = [_p, ctypes.c_int32]
    lib.nesa_trace_name.restype = ctypes.c_char_p
    lib.nesa_ktrace_enable.argtypes = [_p, ctypes.c_int64]
    lib.nesa_ktrace_enable.restype = ctypes.c_int
    lib.nesa_ktrace_read.argtypes = [_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64]
    lib.nesa_ktrace_read.restype = ctypes.c_int64
    lib.nesa_dense_matvec.argtypes = [_p, _p, _p, ctypes.c_int64, ctypes.c_int32, _p]
    lib.nesa_dense_matvec.restype = ctypes.c_int
    lib.nesa_matvec_cols.argtypes = [_p, _p, _p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_uint32, _p]
    lib.nesa_matvec_cols.restype = ctypes.c_int
    lib.nesa_tree_build.argtypes = [_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_void_p)]
    lib.nesa_tree_build.restype = ctypes.c_int
    lib.nesa_tree_error.argtypes = [_p]
    lib.nesa_tree_error.restype = ctypes.c_char_p
    lib.nesa_tree_size.argtypes = [_p, ctypes.c_int32]
    lib.nesa_tree_size.restype = ctypes.c_int64
    lib.nesa_tree_copy.argtypes = [_p, ctypes.c_int32, _p]
    lib.nesa_tree_copy.restype = ctypes.c_int
    lib.nesa_tree_free.argtypes = [_p]
    lib.nesa_tree_free.restype = None
    lib.nesa_exchange_pack.argtypes = [_p, _p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                       ctypes.c_int32, _p, _p]
    lib.nesa_exchange_pack.restype = ctypes.c_int
    lib.nesa_exchange_combine.argtypes = [_p, _p, _p, _p, ctypes.c_int64, ctypes.c_int32,
                                          ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _p]
    lib.nesa_exchange_combine.restype = ctypes.c_int
    lib.nesa_plan_create_dist.argtypes = [ctypes.POINTER(NesaPlanDesc), ctypes.c_int, _p, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.POINTER(NesaExchangeDesc),
                                          ctypes.POINTER(_p)]
    lib.nesa_plan_create_dist.restype = ctypes.c_int
    lib.nesa_nccl_unique_id.argtypes = [_p, ctypes.c_int32]
    lib.nesa_nccl_unique_id.restype = ctypes.c_int
    lib.nesa_nccl_comm_init.argtypes = [_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.POINTER(_p)]
    lib.nesa_nccl_comm_init.restype = ctypes.c_int
    lib.nesa_nccl_comm_destroy.argtypes = [_p]
    lib.nesa_nccl_comm_destroy.restype = ctypes.c_int
    lib.nesa_matvec_near_wide.argtypes = [_p, _p, _p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _p]
    lib.nesa_matvec_near_wide.restype = ctypes.c_int
    lib.nesa_gs_work_bytes.argtypes = []
    lib.nesa_gs_work_bytes.restype = ctypes.c_int64
    lib.nesa_gs_step.argtypes = [_p, ctypes.c_int64, ctypes.c_int32, _p, _p, ctypes.c_int64,
                                 ctypes.c_int32, _p, _p, _p]
    lib.nesa_gs_step.restype = ctypes.c_int
    lib.nesa_gs_step_shifted.argtypes = [_p, ctypes.c_int64, ctypes.c_int32, _p, _p, ctypes.c_int64,
                                         ctypes.c_int32, ctypes.c_double, _p, _p, _p]
    lib.nesa_gs_step_shifted.restype = ctypes.c_int
    lib.nesa_gs_last_error.argtypes = []
    lib.nesa_gs_last_error.restype = ctypes.c_char_p
    if lib.nesa_abi_version() != NESA_ABI_VERSION:
        raise RuntimeError("libnesa_b200.so ABI version mismatch; rebuild")
    _lib = lib
    return lib


class NesaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"nesa error {code}: {msg}")
        self.code = code


def check(code: int) -> None:
    if code != NESA_OK:
        msg = load().nesa_last_error().decode(errors="replace")
        if code in (NESA_ERR_INVALID, NESA_ERR_UNSUPPORTED):
            raise ValueError(msg)
        raise NesaError(code, msg)
