"""ctypes binding of the C ABI in include/absim_gpu.h (libabsim_gpu.so).

There is no fallback: if the sm_100a library is missing or cannot be loaded
this module raises at import time of the engine, and every engine call goes
through the CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ABSIM_GPU_LIB") or os.path.join(HERE, "_lib", "libabsim_gpu.so")

ABS_OK = 0
ABS_ERR_INVALID_ARGUMENT = 1
ABS_ERR_CUDA = 2
ABS_ERR_NONFINITE = 3
ABS_ERR_FIXED_BOX = 4
ABS_ERR_BOX_BUDGET = 5
ABS_ERR_CAPACITY = 6
ABS_ERR_NO_DEVICE = 7
ABS_ERR_STATE = 8

MODEL_NONE, MODEL_PROLIFERATION, MODEL_DRIVE, MODEL_GROW, MODEL_SIR = 0, 1, 2, 3, 4
MODEL_GROW_DIVIDE, MODEL_COHERE = 5, 6  # the reference's own models::GrowDivide / models::Cohere
MODEL_GROW_DIVIDE_DIE = 7  # models::GrowDivide + AgentContext::remove_self with probability mp[3]
FLAG_GHOST = 128
ENV_UNIFORM_GRID, ENV_BRUTE_FORCE, ENV_KD_TREE = 0, 1, 2  # EnvironmentKind (params.hpp:9)

# every symbol include/absim_gpu.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "abs_gpu_default_config", "abs_gpu_create", "abs_gpu_destroy", "abs_gpu_last_error",
    "abs_gpu_upload", "abs_gpu_upload_device", "abs_gpu_set_grid_override", "abs_gpu_local_bounds",
    "abs_gpu_set_iteration", "abs_gpu_sir_counts", "abs_gpu_sir_state",
    "abs_gpu_export_layers", "abs_gpu_import", "abs_gpu_drop_ghosts", "abs_gpu_simulate", "abs_gpu_stats",
    "abs_gpu_synchronize", "abs_gpu_download", "abs_gpu_env_update", "abs_gpu_grid_info",
    "abs_gpu_cell_ids", "abs_gpu_neighbors", "abs_gpu_sort", "abs_gpu_remove",
    "abs_gpu_stream", "abs_gpu_set_stream", "abs_gpu_force_kernel_time", "abs_gpu_reset_timers",
    "abs_gpu_set_defer_commit", "abs_gpu_division_marks", "abs_gpu_commit",
    "abs_gpu_set_agent_ext", "abs_gpu_download_ext", "abs_gpu_phase_times", "abs_gpu_run_frames",
    "abs_gpu_list_stats", "abs_gpu_record_evaluations", "abs_gpu_download_evaluations",
    "abs_gpu_download_storage_keys",
    "abs_gpu_nccl_unique_id", "abs_gpu_comm_init", "abs_gpu_comm_set_transport", "abs_gpu_comm_reserve",
    "abs_gpu_simulate_decomposed", "abs_gpu_decomp_info", "abs_gpu_memcpy",
]

DT_F64_MAX, DT_U64_SUM, DT_U32_SUM = 0, 1, 2

ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p)
COUNTS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                        C.c_void_p)
RECORDS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                         C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p)


class Transport(C.Structure):
    """abs_gpu_transport: caller-side collectives of the slab decomposition."""
    _fields_ = [("user", C.c_void_p), ("allreduce", ALLREDUCE_FN), ("counts", COUNTS_FN), ("records", RECORDS_FN)]


class Config(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("simulation_time_step", C.c_double),
        ("repulsion_coefficient", C.c_double),
        ("max_displacement", C.c_double),
        ("force_threshold", C.c_double),
        ("fixed_box_length", C.c_double),
        ("sorting_frequency", C.c_uint64),
        ("detect_static_agents", C.c_int32),
        ("model", C.c_int32),
        ("model_params", C.c_double * 8),
        ("capacity", C.c_uint64),
        ("record_forces", C.c_int32),
        ("bins_per_box", C.c_int32),
        ("bins_per_box_x", C.c_int32),
        ("environment", C.c_int32),
        ("neighbor_list", C.c_int32),
        ("neighbor_skin", C.c_double),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("agents", C.c_uint64),
        ("uid_count", C.c_uint64),
        ("iterations", C.c_uint64),
        ("force_evaluations", C.c_uint64),
        ("force_skips", C.c_uint64),
        ("agents_added", C.c_uint64),
        ("agents_removed", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("agent_iterations", C.c_uint64),
    ]


class Frame(C.Structure):
    """abs_frame: one host frame of abs_gpu_run_frames."""
    _fields_ = [
        ("n", C.c_uint64),
        ("x", C.POINTER(C.c_double)), ("y", C.POINTER(C.c_double)),
        ("z", C.POINTER(C.c_double)), ("d", C.POINTER(C.c_double)),
        ("out_x", C.POINTER(C.c_double)), ("out_y", C.POINTER(C.c_double)),
        ("out_z", C.POINTER(C.c_double)),
        ("out_cap", C.c_uint64),
        ("n_out", C.POINTER(C.c_uint64)),
        ("out_uid", C.POINTER(C.c_uint64)),
    ]


_D = C.POINTER(C.c_double)
_U64 = C.POINTER(C.c_uint64)
_U32 = C.POINTER(C.c_uint32)
_U8 = C.POINTER(C.c_uint8)
_CTX = C.c_void_p

_lib = None


def load():
    """Load libabsim_gpu.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    sig = {
        "abs_gpu_default_config": (None, [C.POINTER(Config)]),
        "abs_gpu_create": (C.c_int, [C.POINTER(Config), C.c_int, C.POINTER(_CTX)]),
        "abs_gpu_destroy": (C.c_int, [_CTX]),
        "abs_gpu_last_error": (C.c_char_p, [_CTX]),
        "abs_gpu_upload": (C.c_int, [_CTX, C.c_uint64, _U64, _D, _D, _D, _D, _U8, _D, _U8, _U32,
                                     C.c_uint64]),
        "abs_gpu_upload_device": (C.c_int, [_CTX, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]),
        "abs_gpu_set_grid_override": (C.c_int, [_CTX, _D, _U32]),
        "abs_gpu_local_bounds": (C.c_int, [_CTX, _D]),
        "abs_gpu_set_iteration": (C.c_int, [_CTX, C.c_uint64]),
        "abs_gpu_sir_counts": (C.c_int, [_CTX, _U64]),
        "abs_gpu_export_layers": (C.c_int, [_CTX, _D, _U32, C.c_int64, C.c_int64, C.c_int, C.c_void_p,
                                            C.c_void_p, C.c_uint64, _U64, _U64]),
        "abs_gpu_import": (C.c_int, [_CTX, C.c_void_p, C.c_uint64, C.c_int]),
        "abs_gpu_drop_ghosts": (C.c_int, [_CTX]),
        "abs_gpu_set_defer_commit": (C.c_int, [_CTX, C.c_int]),
        "abs_gpu_division_marks": (C.c_int, [_CTX, C.c_void_p, C.c_uint64, _U64]),
        "abs_gpu_commit": (C.c_int, [_CTX, C.c_void_p, C.c_uint64]),
        "abs_gpu_set_agent_ext": (C.c_int, [_CTX, _U32, _U64]),
        "abs_gpu_download_ext": (C.c_int, [_CTX, _U32, _U64]),
        "abs_gpu_phase_times": (C.c_int, [_CTX, _D, _D, C.c_uint64, _U64]),
        "abs_gpu_sir_state": (C.c_int, [_CTX, _U8, _U32]),
        "abs_gpu_run_frames": (C.c_int, [_CTX, C.POINTER(Frame), C.c_uint64, C.c_uint64, C.c_uint64]),
        "abs_gpu_simulate": (C.c_int, [_CTX, C.c_uint64]),
        "abs_gpu_stats": (C.c_int, [_CTX, C.POINTER(Stats)]),
        "abs_gpu_synchronize": (C.c_int, [_CTX]),
        "abs_gpu_download": (C.c_int, [_CTX, _U64, _U64, _D, _D, _D, _D, _D, _D, _D, _U32, _U8, _D]),
        "abs_gpu_env_update": (C.c_int, [_CTX]),
        "abs_gpu_grid_info": (C.c_int, [_CTX, _D, _U32]),
        "abs_gpu_cell_ids": (C.c_int, [_CTX, _U64]),
        "abs_gpu_neighbors": (C.c_int, [_CTX, _U64, _U64, C.c_uint64, _U64]),
        "abs_gpu_sort": (C.c_int, [_CTX]),
        "abs_gpu_remove": (C.c_int, [_CTX, _U64, C.c_uint64]),
        "abs_gpu_stream": (C.c_void_p, [_CTX]),
        "abs_gpu_set_stream": (C.c_int, [_CTX, C.c_void_p]),
        "abs_gpu_force_kernel_time": (C.c_int, [_CTX, _D, _U64]),
        "abs_gpu_reset_timers": (C.c_int, [_CTX, C.c_int]),
        "abs_gpu_list_stats": (C.c_int, [_CTX, _U64, _D]),
        "abs_gpu_record_evaluations": (C.c_int, [_CTX, C.c_int]),
        "abs_gpu_download_evaluations": (C.c_int, [_CTX, _U32, C.c_uint64]),
        "abs_gpu_download_storage_keys": (C.c_int, [_CTX, _U32, C.c_uint64]),
        "abs_gpu_nccl_unique_id": (C.c_int, [C.c_void_p]),
        "abs_gpu_comm_init": (C.c_int, [_CTX, C.c_void_p, C.c_int, C.c_int]),
        "abs_gpu_comm_set_transport": (C.c_int, [_CTX, C.POINTER(Transport), C.c_int, C.c_int]),
        "abs_gpu_comm_reserve": (C.c_int, [_CTX, C.c_uint64]),
        "abs_gpu_simulate_decomposed": (C.c_int, [_CTX, C.c_uint64]),
        "abs_gpu_decomp_info": (C.c_int, [_CTX, C.POINTER(C.c_int64), _U64]),
        "abs_gpu_memcpy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class AbsimError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def check(rc: int, ctx=None):
    """Map a status code to the reference's exception kinds (params.cpp:44-72,
    uniform_grid.cpp:112-141): invalid_argument -> ValueError, others ->
    RuntimeError subclasses carrying the code."""
    if rc == ABS_OK:
        return
    msg = load().abs_gpu_last_error(ctx).decode(errors="replace")
    if rc == ABS_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise AbsimError(rc, msg)
