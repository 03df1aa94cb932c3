"""ctypes binding of libsbg.so (include/sbg.h). The product path has no CPU fallback: if the
library or a GPU is missing, operator construction raises."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SBG_LIB_PATH", os.path.join(_HERE, "libsbg.so"))  # override: A/B builds

SBG_OK, SBG_EINVAL, SBG_ENONCONV, SBG_EDEVICE, SBG_ERUNTIME = 0, 1, 2, 3, 4
SBG_MAX_ROOTS = 64


class Excitation(C.Structure):
    """sbg_excitation == sbci::fci::Excitation (fci/sigma.hpp:19-23)."""
    _fields_ = [("p", C.c_uint16), ("q", C.c_uint16), ("target", C.c_uint32), ("sign", C.c_double)]


class Config(C.Structure):
    _fields_ = [("eps0", C.c_double), ("r0", C.c_double), ("b_th", C.c_double), ("eps1", C.c_double),
                ("x_th1", C.c_double), ("x_th2", C.c_double), ("r1", C.c_double), ("max_cycle", C.c_int32),
                ("hx_refresh_restarts", C.c_int32), ("t_max", C.c_int64), ("lindep", C.c_double),
                ("clamp_delta", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("nroots", C.c_int32), ("iterations", C.c_int32 * SBG_MAX_ROOTS),
                ("restarts", C.c_int32 * SBG_MAX_ROOTS), ("final_residual", C.c_double * SBG_MAX_ROOTS),
                ("matvecs", C.c_uint64), ("total_iterations", C.c_int64), ("total_restarts", C.c_int32),
                ("hx_refreshes", C.c_int32), ("peak_vectors", C.c_int32), ("wall_time_s", C.c_double),
                ("failed_state", C.c_int32), ("best_energy", C.c_double), ("best_residual", C.c_double),
                ("sigma_seconds", C.c_double), ("kernel_launches", C.c_uint64),
                ("s_squared", C.c_double * SBG_MAX_ROOTS), ("device_vectors_peak", C.c_int32)]


class TraceRecordC(C.Structure):
    _fields_ = [("state", C.c_int32), ("t", C.c_int32), ("energy", C.c_double), ("dE", C.c_double),
                ("res_norm", C.c_double), ("x_norm", C.c_double), ("kinetic", C.c_double),
                ("matvecs", C.c_uint64), ("restart_reason", C.c_int32), ("b", C.c_double), ("c", C.c_double),
                ("method", C.c_int32), ("pair_partner", C.c_int32),
                ("b_ab", C.c_double), ("b_ba", C.c_double), ("b_bb", C.c_double), ("c_ab", C.c_double),
                ("c_ba", C.c_double), ("c_bb", C.c_double), ("a_ab", C.c_double), ("a_ba", C.c_double),
                ("energy_partner", C.c_double), ("x_norm_partner", C.c_double), ("res_norm_partner", C.c_double)]


TRACE_FN = C.CFUNCTYPE(None, C.POINTER(TraceRecordC), C.c_void_p)

_lib = None


def lib() -> C.CDLL:
    """Load libsbg.so once. Raises (never falls back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libsbg.so not built ({LIB_PATH}); run `python -m paper_2603_06101_b200.build`")
    L = C.CDLL(LIB_PATH)
    D, P = C.POINTER(C.c_double), C.c_void_p
    sig = {
        "sbg_last_error": (C.c_char_p, []),
        "sbg_version": (C.c_char_p, []),
        "sbg_binomial": (C.c_uint64, [C.c_int, C.c_int]),
        "sbg_ab_plan_info": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64)]),
        "sbg_determinant_count": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64)]),
        "sbg_config_default": (Config, []),
        "sbg_config_validate": (C.c_int, [C.POINTER(Config)]),
        "sbg_synthetic_integrals": (C.c_int, [C.c_int, C.c_uint64, C.c_double, D, D]),
        "sbg_shard_range": (C.c_int, [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "sbg_device_count": (C.c_int, []),
        "sbg_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, D, D, C.c_int, C.c_uint64, C.POINTER(P)]),
        "sbg_create_dist": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, D, D, C.c_int, C.c_uint64, C.c_int,
                                      C.c_int, P, C.POINTER(P)]),
        "sbg_nccl_unique_id": (C.c_int, [P]),
        "sbg_destroy": (None, [P]),
        "sbg_dim": (C.c_int64, [P]),
        "sbg_sector": (C.c_int, [P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "sbg_local_rows": (C.c_int, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "sbg_diagonal": (C.c_int, [P, D]),
        "sbg_table_sizes": (C.c_int, [P, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "sbg_string_tables": (C.c_int, [P, C.c_int, C.POINTER(C.c_uint64), C.POINTER(Excitation)]),
        "sbg_sigma": (C.c_int, [P, D, D, C.c_int]),
        "sbg_sigma_device": (C.c_int, [P, P, P, P]),
        "sbg_padded_len": (C.c_int64, [P]),
        "sbg_pack": (C.c_int, [P, P, P, P]),
        "sbg_unpack": (C.c_int, [P, P, P, P]),
        "sbg_sigma_padded": (C.c_int, [P, P, P, P]),
        "sbg_sigma_padded_multi": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(P), P]),
        "sbg_apply_count": (C.c_uint64, [P]),
        "sbg_reset_apply_count": (None, [P]),
        "sbg_kernel_launches": (C.c_uint64, [P]),
        "sbg_sigma_flops": (C.c_int, [P, D, D, D]),
        "sbg_profile_reset": (C.c_int, [P]),
        "sbg_profile_read": (C.c_int, [P, D, C.POINTER(C.c_int64)]),
        "sbg_spin_squared": (C.c_int, [P, D, D]),
        "sbg_local_group_create": (C.c_int, [C.c_int, C.POINTER(P)]),
        "sbg_local_group_destroy": (None, [P]),
        "sbg_create_local": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, D, D, C.c_int, C.c_uint64, P, C.c_int,
                                       C.POINTER(P)]),
        "sbg_spin_squared_padded": (C.c_int, [P, P, D]),
        "sbg_solve": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(Config), D, D, C.POINTER(Stats), TRACE_FN, P]),
        "sbg_solve_davidson": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(Config), D, D, C.POINTER(Stats), TRACE_FN,
                                         P]),
        "sbg_solve_state_sbci1": (C.c_int, [P, D, C.c_double, D, C.c_int, C.c_int, D, D, D, C.POINTER(Config), D, D,
                                            D, C.POINTER(Stats), TRACE_FN, P]),
        "sbg_selftest": (C.c_int, []),
        "sbg_selftest_nccl": (C.c_int, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


# every symbol declared in include/sbg.h (checked by tests/test_abi.py against the header)
EXPORTED = ["sbg_last_error", "sbg_version", "sbg_binomial", "sbg_ab_plan_info", "sbg_determinant_count", "sbg_config_default",
            "sbg_config_validate", "sbg_synthetic_integrals", "sbg_shard_range", "sbg_device_count", "sbg_create",
            "sbg_create_dist", "sbg_nccl_unique_id", "sbg_destroy", "sbg_dim", "sbg_sector", "sbg_local_rows",
            "sbg_diagonal", "sbg_table_sizes", "sbg_string_tables", "sbg_sigma", "sbg_sigma_device",
            "sbg_padded_len", "sbg_pack", "sbg_unpack", "sbg_sigma_padded", "sbg_sigma_padded_multi", "sbg_apply_count",
            "sbg_reset_apply_count", "sbg_kernel_launches", "sbg_sigma_flops", "sbg_profile_reset", "sbg_profile_read",
            "sbg_spin_squared", "sbg_spin_squared_padded", "sbg_local_group_create", "sbg_local_group_destroy",
            "sbg_create_local", "sbg_solve", "sbg_solve_davidson", "sbg_solve_state_sbci1", "sbg_selftest",
            "sbg_selftest_nccl"]


class SbgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def check(rc: int):
    """Maps library codes onto the reference's exception classes."""
    if rc == SBG_OK:
        return
    msg = lib().sbg_last_error().decode()
    if rc == SBG_EINVAL:
        raise ValueError(msg)          # std::invalid_argument
    if rc == SBG_ERUNTIME:
        raise SbgError(rc, msg)        # std::runtime_error
    if rc == SBG_ENONCONV:
        from .solver import NonConvergenceError
        raise NonConvergenceError(msg)
    raise SbgError(rc, msg)
