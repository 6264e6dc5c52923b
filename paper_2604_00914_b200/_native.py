"""Loader for libadp_b200.so (the C-ABI in include/adp.h).

The product path has no fallback: if the shared library is missing or cannot
be loaded, every entry point raises. Build it with ``__graft_entry__.build()``
(or ``make -C paper_2604_00914_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libadp_b200.so")

# adp_status codes -> exception types mirroring the reference's
# (proj/include/adapoly/types.hpp:23-46).
ADP_OK, ADP_ERR_CONFIG, ADP_ERR_DIMENSION, ADP_ERR_NOT_PD, ADP_ERR_PARSE = 0, 1, 2, 3, 4
ADP_ERR_RUNTIME, ADP_ERR_CUDA, ADP_ERR_OOM, ADP_ERR_NCCL = 5, 6, 7, 8
ADP_F64, ADP_C128 = 0, 1
ADP_COL_MAJOR, ADP_ROW_MAJOR = 0, 1


class AdpError(RuntimeError):
    code = ADP_ERR_RUNTIME


class ConfigError(AdpError, ValueError):
    code = ADP_ERR_CONFIG


class DimensionError(AdpError, ValueError):
    code = ADP_ERR_DIMENSION


class NotPositiveDefinite(AdpError):
    code = ADP_ERR_NOT_PD


class ParseError(AdpError):
    code = ADP_ERR_PARSE


class CudaError(AdpError):
    code = ADP_ERR_CUDA


class OutOfMemory(CudaError):
    code = ADP_ERR_OOM


class CollectiveError(AdpError):
    code = ADP_ERR_NCCL


_EXC = {c.code: c for c in (ConfigError, DimensionError, NotPositiveDefinite, ParseError, CudaError, OutOfMemory,
                            CollectiveError)}


class FilterInfo(C.Structure):
    """adp_filter_info (ChebFilter minus coeffs, cheb_filter.hpp:41-66)."""

    _fields_ = [
        ("interval_a", C.c_double), ("interval_b", C.c_double),
        ("alpha", C.c_double), ("beta", C.c_double),
        ("k_max", C.c_int32), ("m", C.c_double), ("l1", C.c_double), ("l2", C.c_double),
        ("lambda_min", C.c_double), ("lambda_max", C.c_double), ("active_degree", C.c_int32),
    ]


class HaloTarget(C.Structure):
    """adp_halo_target: a neighbour's rows of a halo-extended block (peer memory)."""

    _fields_ = [("dst", C.c_void_p), ("row_lo", C.c_int64), ("row_hi", C.c_int64), ("row_shift", C.c_int64),
                ("ld", C.c_int64)]


P, I32, I64, U64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double

# name -> (restype, argtypes); every symbol declared in include/adp.h.
SIGNATURES = {
    "adp_version": (I32, []),
    "adp_last_error_message": (C.c_char_p, []),
    "adp_ctx_create": (I32, [I32, P]),
    "adp_ctx_destroy": (I32, [P]),
    "adp_ctx_set_stream": (I32, [P, P]),
    "adp_ctx_own_stream": (P, [P]),
    "adp_ctx_synchronize": (I32, [P]),
    "adp_ctx_launch_count": (I64, [P]),
    "adp_ctx_last_step_kernel": (I32, [P]),
    "adp_csr_stencil": (I32, [P, P, P]),
    "adp_spmv_device": (I32, [P, P, P, P]),
    "adp_ctx_set_panel": (I32, [P, I32]),
    "adp_ctx_set_tuning": (I32, [P, I32]),
    "adp_csr_create": (I32, [P, I64, I64, P, P, P, I32, P]),
    "adp_csr_create_device": (I32, [P, I64, I64, I64, P, P, P, I32, P]),
    "adp_csr_destroy": (I32, [P]),
    "adp_csr_info": (I32, [P, P, P, P, P]),
    "adp_filter_apply": (I32, [P, P, P, I32, D, D, I32, P, I64, I64, I64, I32, P, I64, P]),
    "adp_filter_apply_device": (I32, [P, P, P, I32, D, D, I32, P, I64, I64, I64, P, I64, P]),
    "adp_step_device": (I32, [P, P, I32, P, I64, P, P, I64, P, P, I64, I64, I64, I64, I64, D, D, D, D]),
    "adp_step_device_push": (I32, [P, P, I32, P, I64, P, P, I64, P, P, I64, I64, I64, I64, I64, D, D, D, D, P, I32]),
    "adp_halo_push_rows": (I32, [P, I32, P, I64, I64, I64, I64, P, I32]),
    "adp_halo_signal": (I32, [P, P, I32, U64]),
    "adp_halo_wait": (I32, [P, P, I32, U64, C.c_uint32]),
    "adp_halo_check": (I32, [P]),
    "adp_ipc_handle": (I32, [P, P]),
    "adp_ipc_open": (I32, [I32, P, P]),
    "adp_ipc_close": (I32, [P]),
    "adp_spmm": (I32, [P, P, P, I64, I64, I64, I32, P, I64, I32]),
    "adp_spmm_device": (I32, [P, P, P, I64, I64, I64, P, I64, I32]),
    "adp_step_coeffs": (I32, [D, D, I32, P]),
    "adp_lanczos_damping": (I32, [I32, D, P]),
    "adp_jackson_damping": (I32, [I32, P]),
    "adp_build_filter": (I32, [D, D, D, D, I32, D, I32, P, P]),
    "adp_eval_filter": (I32, [P, P, P, I64, I32, P, P]),
    "adp_initial_degree": (I32, [D, D, D, P]),
    "adp_j_theta": (I32, [D, D, D, P]),
    "adp_c_m_constant": (I32, [D, P]),
    "adp_undamped_bound": (I32, [D, I32, D, D, P]),
    "adp_damped_bound": (I32, [D, I32, I32, D, D, D, P]),
    "adp_projector_bound": (I32, [P, P, I64, I32, P]),
    "adp_adaptive_degree": (I32, [P, P, P, I64, I64, D, P]),
    "adp_fill_gaussian": (I32, [P, I64, I64, U64, U64]),
    "adp_fill_rademacher": (I32, [P, I64, I64, U64, U64]),
    "adp_philox_gaussian": (I32, [U64, U64, U64, I64, P]),
    "adp_philox_uniform": (I32, [U64, U64, U64, I64, P]),
    "adp_philox_block": (I32, [U64, U64, U64, P]),
    "adp_fill_gaussian_device": (I32, [P, P, I64, I64, I64, U64, U64]),
    "adp_fill_rademacher_device": (I32, [P, P, I64, I64, I64, U64, U64]),
    "adp_lanczos_bounds": (I32, [P, P, I32, U64, P, P, P]),
    "adp_estimate_eigcount": (I32, [P, P, P, I32, D, D, I64, U64, P, P]),
    "adp_cholesky_qr_device": (I32, [P, P, I64, I64, I64, P]),
    "adp_rayleigh_ritz_device": (I32, [P, P, P, I64, I64, P, P, I64]),
    "adp_residual_norms_device": (I32, [P, P, P, I64, I64, P, P]),
    "adp_spurious_threshold": (I32, [P, I64, D, D, P]),
    "adp_solver_config_default": (None, [P]),
    "adp_solve": (I32, [P, P, P, P]),
    "adp_solve_summary_get": (I32, [P, P]),
    "adp_solve_eigenpairs": (I32, [P, P, P, I64]),
    "adp_solve_history": (I32, [P, P, P]),
    "adp_solve_result_destroy": (I32, [P]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded C-ABI library; raises if it is not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libadp_b200.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != ADP_OK:
        msg = lib().adp_last_error_message().decode(errors="replace")
        raise _EXC.get(status, AdpError)(msg)
