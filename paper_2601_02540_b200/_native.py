"""ctypes binding of the C ABI in include/hsgn_b200.h.

Loads paper_2601_02540_b200/_native/libhsgn_b200.so (built in-tree by
``paper_2601_02540_b200.build``).  There is no fallback: if the library is
missing or cannot be loaded, importing the operators raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HSGN_LIB may point at an alternative in-tree build (A/B measurements of
# kernel variants in one GPU session); default: the in-tree library.
LIB_PATH = os.environ.get("HSGN_LIB") or os.path.join(HERE, "_native", "libhsgn_b200.so")

D = C.c_double
PD = C.POINTER(C.c_double)
I32 = C.c_int32
I64 = C.c_int64

HSGN_OK, HSGN_EINVAL, HSGN_EDEPTH, HSGN_ECUDA, HSGN_ENCCL = range(5)
STATUS_NAMES = {0: "HSGN_OK", 1: "HSGN_EINVAL", 2: "HSGN_EDEPTH", 3: "HSGN_ECUDA", 4: "HSGN_ENCCL"}


class hsgn_grid(C.Structure):
    _fields_ = [("nx", I32), ("ny", I32), ("kind_x", I32), ("kind_y", I32),
                ("x_min", D), ("x_max", D), ("y_min", D), ("y_max", D)]


class hsgn_phys(C.Structure):
    _fields_ = [("g", D), ("lambda_", D), ("h_floor", D)]


class hsgn_cfg(C.Structure):
    _fields_ = [("abs_tol", D), ("rel_tol", D), ("dt_initial", D), ("dt_max", D), ("safety", D),
                ("growth_cap", D), ("shrink_floor", D), ("max_steps", I64), ("fixed_dt", D),
                ("h_floor", D)]


class hsgn_record(C.Structure):
    _fields_ = [("t", D), ("accepted", I64), ("rejected", I64), ("rhs_evals", I64),
                ("rhs_evals_setup", I64), ("aborted", I32), ("reason", C.c_char * 256)]


class hsgn_scenario(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("domain", hsgn_grid), ("g", D), ("lambda_", D), ("t0", D),
                ("t_final", D), ("has_source", I32), ("has_exact", I32), ("n_exact_vars", I32),
                ("exact_vars", I32 * 5), ("n_gauges", I32), ("n_snapshots", I32), ("gauges", (D * 2) * 8),
                ("snapshot_times", D * 8), ("kind", I32), ("reserved", I32), ("p", D * 24)]


CTX = C.c_void_p
STATE = C.c_void_p
OBSERVER = C.CFUNCTYPE(None, D, STATE, STATE, C.c_void_p)

_lib = None


def lib() -> C.CDLL:
    """The loaded native library (built on first use if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

    def f(name, res, *args):
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = list(args)

    G, PH, CF, RC = C.POINTER(hsgn_grid), C.POINTER(hsgn_phys), C.POINTER(hsgn_cfg), C.POINTER(hsgn_record)
    PCTX, PST = C.POINTER(CTX), C.POINTER(STATE)
    f("hsgn_ctx_create", C.c_int, G, PH, PD, C.c_int, PCTX)
    f("hsgn_ctx_create_slab", C.c_int, G, PH, PD, C.c_int, I32, I32, I32, I32, PCTX)
    f("hsgn_nccl_unique_id", C.c_int, C.c_char_p)
    f("hsgn_ctx_attach_nccl", C.c_int, CTX, C.c_char_p)
    f("hsgn_ctx_destroy", C.c_int, CTX)
    f("hsgn_last_error", C.c_char_p, CTX)
    f("hsgn_set_source", C.c_int, CTX, I32)
    f("hsgn_set_rows_per_block", C.c_int, CTX, I32)
    f("hsgn_set_stencil_kind", C.c_int, CTX, I32)
    f("hsgn_stencil_kind", I32, CTX)
    f("hsgn_set_fused_stages", C.c_int, CTX, I32)
    f("hsgn_fused_stages", I32, CTX)
    f("hsgn_profile_fused", C.c_int, CTX, STATE, STATE, D, I32, PD)
    f("hsgn_n_evals", I64, CTX)
    f("hsgn_state_alloc", C.c_int, CTX, PST)
    f("hsgn_state_free", C.c_int, CTX, STATE)
    f("hsgn_state_upload", C.c_int, CTX, STATE, PD)
    f("hsgn_state_download", C.c_int, CTX, STATE, PD)
    f("hsgn_state_copy", C.c_int, CTX, STATE, STATE)
    f("hsgn_state_field_ptr", C.c_int, STATE, I32, C.POINTER(PD))
    f("hsgn_rhs", C.c_int, CTX, D, STATE, STATE, C.POINTER(I64))
    f("hsgn_rhs_shallow_water", C.c_int, CTX, D, STATE, STATE, C.POINTER(I64))
    f("hsgn_init_auxiliary", C.c_int, CTX, STATE)
    f("hsgn_solve", C.c_int, CTX, STATE, D, D, CF, STATE, RC, OBSERVER, C.c_void_p)
    f("hsgn_bs3_fixed_steps", C.c_int, CTX, STATE, STATE, D, D, I64, C.POINTER(I64))
    f("hsgn_prepare_fixed_steps", C.c_int, CTX, STATE, STATE, D, I64)
    f("hsgn_set_kernel_timing", C.c_int, CTX, I32)
    f("hsgn_kernel_times", C.c_int, CTX, PD, PD, C.POINTER(I64))
    f("hsgn_total_mass", C.c_int, CTX, STATE, PD)
    f("hsgn_total_energy", C.c_int, CTX, STATE, PD)
    f("hsgn_energy_rate", C.c_int, CTX, STATE, STATE, PD)
    f("hsgn_mass_weighted_sum", C.c_int, CTX, STATE, I32, PD)
    f("hsgn_discrete_l2_error", C.c_int, CTX, STATE, STATE, I32, PD)
    f("hsgn_row_sums", C.c_int, CTX, I32, STATE, STATE, I32, PD)
    f("hsgn_outer_sum", D, G, PD, I32, I32)
    f("hsgn_synchronize", C.c_int, CTX)
    f("hsgn_last_timing", C.c_int, CTX, PD, C.POINTER(I64))
    f("hsgn_build_info", C.c_char_p)
    f("hsgn_profile_stages", C.c_int, CTX, STATE, STATE, D, I32, PD)
    GRP, GST = C.c_void_p, C.c_void_p
    f("hsgn_group_create", C.c_int, G, PH, PD, C.POINTER(C.c_int), I32, C.POINTER(GRP))
    f("hsgn_group_destroy", C.c_int, GRP)
    f("hsgn_group_last_error", C.c_char_p, GRP)
    f("hsgn_group_state_alloc", C.c_int, GRP, C.POINTER(GST))
    f("hsgn_group_state_free", C.c_int, GRP, GST)
    f("hsgn_group_state_upload", C.c_int, GRP, GST, PD)
    f("hsgn_group_state_download", C.c_int, GRP, GST, PD)
    f("hsgn_group_rhs", C.c_int, GRP, D, GST, GST, C.POINTER(I64))
    f("hsgn_group_bs3_fixed_steps", C.c_int, GRP, GST, GST, D, D, I64, C.POINTER(I64))
    f("hsgn_group_reduce", C.c_int, GRP, I32, GST, GST, PD)
    REC = C.c_void_p
    f("hsgn_recorder_create", C.c_int, CTX, I32, PD, I32, PD, I64, C.POINTER(REC))
    f("hsgn_recorder_destroy", C.c_int, REC)
    f("hsgn_solve_recorded", C.c_int, CTX, STATE, D, D, CF, STATE, RC, OBSERVER, C.c_void_p, REC)
    f("hsgn_recorder_counts", C.c_int, REC, C.POINTER(I64), C.POINTER(I64), C.POINTER(I32))
    f("hsgn_recorder_gauge_node", C.c_int, REC, I32, C.POINTER(I32), C.POINTER(I32), PD, PD)
    f("hsgn_recorder_gauges", C.c_int, REC, PD, PD)
    f("hsgn_recorder_conservation", C.c_int, REC, PD)
    f("hsgn_recorder_snapshot", C.c_int, REC, I32, PD, PD, PD)
    SC = C.POINTER(hsgn_scenario)
    f("hsgn_scenario_count", I32)
    f("hsgn_scenario_name", C.c_char_p, I32)
    f("hsgn_scenario_make", C.c_int, C.c_char_p, C.POINTER(C.c_char_p), PD, I32, SC, C.c_char_p, I32)
    f("hsgn_scenario_sample", C.c_int, SC, I32, I32, PD, PD)
    f("hsgn_scenario_sample_rows", C.c_int, SC, I32, I32, I32, I32, PD, PD)
    f("hsgn_scenario_exact", C.c_int, SC, I32, I32, D, PD)
    f("hsgn_scenario_eval", C.c_int, SC, D, D, PD)
    _lib = L
    return L


# Every exported symbol of include/hsgn_b200.h (checked by tests/test_abi.py).
EXPORTS = [
    "hsgn_ctx_create", "hsgn_ctx_create_slab", "hsgn_nccl_unique_id", "hsgn_ctx_attach_nccl",
    "hsgn_ctx_destroy", "hsgn_last_error", "hsgn_set_source", "hsgn_set_rows_per_block",
    "hsgn_set_stencil_kind", "hsgn_stencil_kind", "hsgn_n_evals",
    "hsgn_state_alloc", "hsgn_state_free", "hsgn_state_upload", "hsgn_state_download", "hsgn_state_copy",
    "hsgn_state_field_ptr", "hsgn_rhs", "hsgn_rhs_shallow_water", "hsgn_init_auxiliary", "hsgn_solve",
    "hsgn_bs3_fixed_steps", "hsgn_total_mass", "hsgn_total_energy", "hsgn_energy_rate",
    "hsgn_mass_weighted_sum", "hsgn_discrete_l2_error", "hsgn_row_sums", "hsgn_outer_sum",
    "hsgn_synchronize", "hsgn_last_timing", "hsgn_build_info", "hsgn_profile_stages",
    "hsgn_group_create", "hsgn_group_destroy", "hsgn_group_last_error", "hsgn_group_state_alloc",
    "hsgn_group_state_free", "hsgn_group_state_upload", "hsgn_group_state_download", "hsgn_group_rhs",
    "hsgn_group_bs3_fixed_steps", "hsgn_group_reduce",
    "hsgn_recorder_create", "hsgn_recorder_destroy", "hsgn_solve_recorded", "hsgn_recorder_counts",
    "hsgn_recorder_gauge_node", "hsgn_recorder_gauges", "hsgn_recorder_conservation", "hsgn_recorder_snapshot",
    "hsgn_set_fused_stages", "hsgn_fused_stages", "hsgn_profile_fused",
    "hsgn_scenario_count", "hsgn_scenario_name", "hsgn_scenario_make", "hsgn_scenario_sample",
    "hsgn_scenario_exact", "hsgn_prepare_fixed_steps", "hsgn_scenario_eval",
    "hsgn_set_kernel_timing", "hsgn_kernel_times", "hsgn_scenario_sample_rows",
]
