"""ctypes binding of the C ABI declared in include/gridtune_cuda.h.

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is deliberately no fallback: if the library is missing or
no CUDA device is usable, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "libgridtune_b200.so"

# status codes (gridtune_cuda.h)
GTC_OK = 0
GTC_ERR_INVALID = -1
GTC_ERR_CONDITIONING = -2
GTC_ERR_NO_CANDIDATES = -3
GTC_ERR_CUDA = -4
GTC_ERR_OOM = -5
GTC_ERR_CONFIG = -6
GTC_ERR_CAPACITY = -7


class gtc_kernel(C.Structure):
    _fields_ = [("nu", C.c_int32), ("lengthscale", C.c_double), ("output_variance", C.c_double)]


class gtc_model_config(C.Structure):
    _fields_ = [("kernel", gtc_kernel), ("noise", C.c_double), ("jitter", C.c_double),
                ("n_max", C.c_int32)]


class gtc_fit_info(C.Structure):
    _fields_ = [("n", C.c_int32), ("rebuilt", C.c_int32), ("y_mean", C.c_double),
                ("y_std", C.c_double), ("jitter", C.c_double)]


class gtc_select_args(C.Structure):
    _fields_ = [("af_mask", C.c_uint32), ("lambda_mode", C.c_int32),
                ("lambda_constant", C.c_double), ("cv_initial_sample_mean", C.c_double),
                ("cv_initial_mean_variance", C.c_double), ("f_best_raw", C.c_double),
                ("excluded", C.POINTER(C.c_int64)), ("n_excluded", C.c_int32)]


class gtc_select_result(C.Structure):
    _fields_ = [("position", C.c_int64 * 3), ("score", C.c_double * 3), ("lambda_", C.c_double),
                ("mean_variance", C.c_double), ("best_std", C.c_double),
                ("n_candidates", C.c_int64), ("cv_fallback", C.c_int32)]


class gtc_step_record(C.Structure):
    _fields_ = [("position", C.c_int64), ("value", C.c_double), ("lambda_", C.c_double),
                ("valid", C.c_int32), ("cv_fallback", C.c_int32), ("by", C.c_int32), ("pad", C.c_int32)]


class gtc_portfolio_config(C.Structure):
    _fields_ = [("mode", C.c_int32), ("skip_threshold", C.c_int32), ("discount", C.c_double),
                ("required_improvement", C.c_double)]


class gtc_portfolio_op(C.Structure):
    _fields_ = [("kind", C.c_int32), ("af", C.c_int32), ("picks", C.c_int64 * 3), ("value", C.c_double)]


class gtc_portfolio_state(C.Structure):
    _fields_ = [("position", C.c_int64), ("by", C.c_int32), ("active", C.c_int32 * 3),
                ("duplicates", C.c_int32 * 3), ("above", C.c_int32 * 3), ("below", C.c_int32 * 3),
                ("pad", C.c_int32), ("dos", C.c_double * 3)]


GTC_STEPS_HOLD_N = 1
GTC_STEPS_TIMING = 2


class gtc_shard_selection(C.Structure):
    _fields_ = [("best_position", C.c_int64 * 3), ("best_score", C.c_double * 3),
                ("first_eligible", C.c_int64), ("first_nan_mask", C.c_uint32),
                ("n_candidates", C.c_int64), ("lambda_", C.c_double), ("mean_variance", C.c_double),
                ("best_std", C.c_double), ("cv_fallback", C.c_int32)]


class gtc_bo_config(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("seed", C.c_uint64), ("budget", C.c_int64),
                ("n_init", C.c_int64), ("invalid_consumes_budget", C.c_int32), ("nu", C.c_int32),
                ("lengthscale", C.c_double), ("output_variance", C.c_double), ("noise", C.c_double),
                ("jitter", C.c_double), ("exploration_mode", C.c_int32),
                ("exploration_constant", C.c_double), ("discount", C.c_double),
                ("required_improvement", C.c_double), ("skip_threshold", C.c_int32),
                ("lhs_restarts", C.c_int64)]


class gtc_bo_record(C.Structure):
    _fields_ = [("position", C.c_int64), ("id", C.c_uint64), ("value", C.c_double),
                ("valid", C.c_int32), ("best_so_far", C.c_double)]


class gtc_bo_summary(C.Structure):
    _fields_ = [("evaluations", C.c_int64), ("budget_consumed", C.c_int64),
                ("invalid_count", C.c_int64), ("surrogate_size", C.c_int64),
                ("n_records", C.c_int64), ("n_lambdas", C.c_int64), ("best_position", C.c_int64),
                ("best_value", C.c_double), ("n_warnings", C.c_int32)]


P = C.c_void_p
DP = C.POINTER(C.c_double)
I64P = C.POINTER(C.c_int64)
U64P = C.POINTER(C.c_uint64)
U8P = C.POINTER(C.c_uint8)
OBJECTIVE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_uint64, DP)

GTC_ERR_SAMPLING = -8
GTC_ERR_ABORTED = -9
GTC_ERR_PARSE = -10
GTC_ERR_EMPTY = -11


class gtc_param_def(C.Structure):
    _fields_ = [("name", C.c_char_p), ("kind", C.c_int32), ("n_values", C.c_int32),
                ("numbers", C.POINTER(C.c_double)), ("strings", C.POINTER(C.c_char_p)),
                ("booleans", C.POINTER(C.c_uint8))]

# (name, restype, argtypes) — exactly the declarations of include/gridtune_cuda.h
SIGNATURES = [
    ("gtc_last_error", C.c_char_p, []),
    ("gtc_version", C.c_char_p, []),
    ("gtc_kernel_launches", C.c_uint64, []),
    ("gtc_space_create", C.c_int, [C.c_int, DP, C.c_int64, C.c_int32, C.POINTER(P)]),
    ("gtc_space_destroy", C.c_int, [P]),
    ("gtc_space_size", C.c_int64, [P]),
    ("gtc_space_enumerate", C.c_int, [C.c_int, C.POINTER(gtc_param_def), C.c_int32, C.POINTER(C.c_char_p),
                                      C.c_int32, I64P, C.POINTER(P)]),
    ("gtc_space_ids", C.c_int, [P, U64P]),
    ("gtc_space_cartesian_size", C.c_uint64, [P]),
    ("gtc_space_nearest", C.c_int, [P, DP, C.c_int32, I64P]),
    ("gtc_restriction_validate", C.c_int, [C.POINTER(gtc_param_def), C.c_int32, C.c_char_p, I64P]),
    ("gtc_run_create", C.c_int, [P, C.POINTER(gtc_model_config), C.POINTER(P)]),
    ("gtc_run_destroy", C.c_int, [P]),
    ("gtc_run_reset", C.c_int, [P, C.POINTER(gtc_model_config)]),
    ("gtc_run_acquire", C.c_int, [P, C.POINTER(gtc_model_config), C.POINTER(P)]),
    ("gtc_run_release", C.c_int, [P]),
    ("gtc_fit", C.c_int, [P, I64P, DP, C.c_int32, C.POINTER(gtc_fit_info)]),
    ("gtc_append", C.c_int, [P, C.c_int64, C.c_double, C.POINTER(gtc_fit_info)]),
    ("gtc_truncate", C.c_int, [P, C.c_int32, C.POINTER(gtc_fit_info)]),
    ("gtc_mark_visited", C.c_int, [P, C.c_int64]),
    ("gtc_unmark_visited", C.c_int, [P, C.c_int64]),
    ("gtc_unvisited_count", C.c_int64, [P]),
    ("gtc_select", C.c_int, [P, C.POINTER(gtc_select_args), C.POINTER(gtc_select_result)]),
    ("gtc_observe", C.c_int, [P, C.c_int64, C.c_double, C.c_int32, C.POINTER(gtc_select_args),
                              C.POINTER(gtc_select_result), C.POINTER(gtc_fit_info)]),
    ("gtc_run_set_values", C.c_int, [P, DP, C.c_int64]),
    ("gtc_run_set_portfolio", C.c_int, [P, C.POINTER(gtc_portfolio_config)]),
    ("gtc_run_set_pdl", C.c_int, [P, C.c_int32]),
    ("gtc_portfolio_trace", C.c_int, [C.c_int, C.POINTER(gtc_portfolio_config), C.POINTER(C.c_int32), C.c_int32,
                                      C.POINTER(gtc_portfolio_op), C.POINTER(gtc_portfolio_state)]),
    ("gtc_run_steps", C.c_int, [P, C.POINTER(gtc_select_args), C.c_int32, C.c_int32,
                                C.POINTER(gtc_step_record), C.POINTER(C.c_int32), C.POINTER(gtc_fit_info)]),
    ("gtc_last_steps_ms", C.c_double, [P]),
    ("gtc_last_steps_phase_ms", C.c_int, [P, DP]),
    ("gtc_mean_variance", C.c_int, [P, DP, I64P]),
    ("gtc_read_predictions", C.c_int, [P, DP, DP]),
    ("gtc_last_pass_ms", C.c_double, [P]),
    ("gtc_last_step_ms", C.c_double, [P]),
    ("gtc_debug_append_marks", C.c_int, [P, U64P]),
    ("gtc_last_phase_ms", C.c_int, [P, DP]),
    ("gtc_run_stream", C.c_uint64, [P]),
    ("gtc_run_exact_rows", C.c_int64, [P]),
    ("gtc_debug_select_trace", C.c_int, [U64P, C.c_int32]),
    ("gtc_debug_set_rebuild", C.c_int, [C.c_int32]),
    ("gtc_debug_set_factor", C.c_int, [C.c_int32]),
    ("gtc_gp_fit", C.c_int, [C.c_int, C.POINTER(gtc_kernel), DP, DP, C.c_int32, C.c_int32,
                             C.c_double, C.c_double, C.POINTER(P), C.POINTER(gtc_fit_info)]),
    ("gtc_gp_predict", C.c_int, [P, DP, C.c_int64, DP, DP]),
    ("gtc_gp_info", C.c_int, [P, C.POINTER(gtc_fit_info)]),
    ("gtc_gp_destroy", C.c_int, [P]),
    ("gtc_best_candidate", C.c_int, [C.c_int, C.c_int32, DP, DP, C.c_int64, C.c_double,
                                     C.c_double, U8P, I64P, DP]),
    ("gtc_acquisition_scores", C.c_int, [C.c_int, C.c_int32, DP, DP, C.c_int64, C.c_double,
                                         C.c_double, DP]),
    ("gtc_fit_points", C.c_int, [P, DP, DP, C.c_int32, C.POINTER(gtc_fit_info)]),
    ("gtc_run_set_shard", C.c_int, [P, C.c_int64]),
    ("gtc_shard_observe", C.c_int, [P, DP, C.c_int64, C.c_double, C.c_int32, DP, I64P,
                                    C.POINTER(gtc_fit_info)]),
    ("gtc_shard_select", C.c_int, [P, C.POINTER(gtc_select_args), C.c_double, C.c_int64,
                                   C.POINTER(gtc_shard_selection)]),
    ("gtc_space_coords", DP, [P]),
    ("gtc_space_dimension", C.c_int32, [P]),
    ("gtc_space_device", C.c_int32, [P]),
    ("gtc_run_bo", C.c_int, [P, U64P, C.POINTER(gtc_bo_config), OBJECTIVE_FN, C.c_void_p,
                             C.POINTER(gtc_bo_record), DP, C.c_int64, C.POINTER(gtc_bo_summary)]),
    ("gtc_run_bo_table", C.c_int, [P, U64P, C.POINTER(gtc_bo_config), DP, C.POINTER(gtc_bo_record), DP,
                                   C.c_int64, C.POINTER(gtc_bo_summary)]),
    ("gtc_group_create", C.c_int, [C.c_int, C.POINTER(P)]),
    ("gtc_group_destroy", C.c_int, [P]),
    ("gtc_group_join", C.c_int, [P]),
    ("gtc_group_leave", C.c_int, [P]),
    ("gtc_run_set_group", C.c_int, [P, P]),
    ("gtc_cache_checksum", C.c_uint64, [U64P, DP, U8P, C.c_int64]),
    ("gtc_comm_nccl_id", C.c_int, [U8P]),
    ("gtc_comm_create_nccl", C.c_int, [U8P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(P)]),
    ("gtc_comm_wrap_nccl", C.c_int, [C.c_void_p, C.POINTER(P)]),
    ("gtc_comm_create_local", C.c_int, [C.c_int32, C.POINTER(P)]),
    ("gtc_comm_destroy", C.c_int, [P]),
    ("gtc_comm_rank", C.c_int32, [P]),
    ("gtc_comm_size", C.c_int32, [P]),
    ("gtc_run_attach_comm", C.c_int, [P, P, C.c_int64, C.c_int64]),
    ("gtc_run_bo_batch", C.c_int, [P, U64P, C.POINTER(gtc_bo_config), C.c_int32, DP, C.c_int32,
                                   C.POINTER(gtc_bo_record), DP, C.c_int64, C.POINTER(gtc_bo_summary),
                                   C.POINTER(C.c_int32)]),
]

_lib = None


def load() -> C.CDLL:
    """Loads libgridtune_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("GRIDTUNE_B200_LIB", str(LIB_PATH))
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().gtc_last_error().decode()


def dptr(a):
    return a.ctypes.data_as(DP)


def i64ptr(a):
    return a.ctypes.data_as(I64P)


def u8ptr(a):
    return a.ctypes.data_as(U8P)
