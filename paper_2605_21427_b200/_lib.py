"""Loader for libpals_gpu.so — the only compute path of this package.

There is no CPU fallback: if the library is missing or no sm_100 device is
visible, every entry point raises. ``load()`` builds the library in-tree when
the .so is absent (nvcc cross-compiles without a GPU).
"""
from __future__ import annotations

import ctypes as C
import os

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
# PALS_GPU_LIB: an alternative in-tree build of the same library (kernel A/B variants)
LIB_PATH = os.environ.get("PALS_GPU_LIB") or os.path.join(_HERE, "libpals_gpu.so")

_VP = C.c_void_p
_I = C.c_int
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double

# (name, restype, argtypes) for every symbol declared in include/pals_gpu.h
SIGNATURES = [
    ("pals_last_error", C.c_char_p, []),
    ("pals_abi_version", _I, []),
    ("pals_ctx_create", _I, [_I, _VP]),
    ("pals_ctx_destroy", _I, [_VP]),
    ("pals_ctx_set_stream", _I, [_VP, _VP]),
    ("pals_ctx_stream", _VP, [_VP]),
    ("pals_ctx_sync", _I, [_VP]),
    ("pals_ctx_launch_count", _I64, [_VP]),
    ("pals_ctx_set_replay_layout", _I, [_VP, C.c_int32]),
    ("pals_ctx_set_one_server", _I, [_VP, C.c_int64]),
    ("pals_model_analytic", _I, [_VP, _VP, _VP, _VP]),
    ("pals_model_table", _I, [_VP, _VP, _VP, _VP, _I64, _VP]),
    ("pals_model_forest", _I, [_VP, _I32, _I32, _VP,
                               _I32, _VP, _VP, _VP, _VP, _VP, _VP,
                               _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    ("pals_model_destroy", _I, [_VP]),
    ("pals_model_forest_cells", _I64, [_VP]),
    ("pals_model_forest_set_direct", _I, [_VP, _I]),
    ("pals_eval_device", _I, [_VP, _VP, _VP, _VP, _VP]),
    ("pals_predict_device", _I, [_VP, _VP, _VP, _I64, _VP, _VP]),
    ("pals_grid_points", _I, [_VP, _VP, _I64, _VP]),
    ("pals_grid_axes", _I, [_VP, _VP, _I32, _VP, _I32, _VP, _I32, _VP, _I32, _VP, _I32, _VP]),
    ("pals_grid_size", _I64, [_VP]),
    ("pals_grid_destroy", _I, [_VP]),
    ("pals_eval", _I, [_VP, _VP, _VP, _VP, _VP]),
    ("pals_plan_create", _I, [_VP, _VP, _VP, _VP, _VP]),
    ("pals_plan_destroy", _I, [_VP]),
    ("pals_plan_prepare", _I, [_VP]),
    ("pals_plan_select_device", _I, [_VP, _VP, _I64, _VP, _VP]),
    ("pals_select", _I, [_VP, _VP, _I64, _VP, _VP]),
    ("pals_plan_run", _I, [_VP, _VP, _I64, _VP, _VP]),
    ("pals_plan_scores", _I, [_VP, _VP, _VP, _VP]),
    ("pals_plan_last_exact_count", _I64, [_VP]),
    ("pals_plan_set_force_exact", _I, [_VP, _I]),
    ("pals_plan_set_decide", _I, [_VP, _I32]),
    ("pals_plan_stats", _I, [_VP, _VP]),
    ("pals_plan_time_scan", _I, [_VP, _I]),
    ("pals_plan_scan_ms", _D, [_VP]),
    ("pals_measure_peaks", _I, [_VP, _VP, _VP]),
    ("pals_select_one", _I, [_VP, _VP, _VP, _I64, _VP, _VP, _D, _D, _D, _VP]),
    ("pals_control_step_one", _I, [_VP, _VP, _VP, _D, _VP, _VP, _I64, _VP, _VP, _VP, _VP,
                                   _VP]),
    ("pals_replay", _I, [_VP, _I32, _VP, _VP, _VP, _VP, _VP, _I32, _VP, _I32, _VP, _VP, _VP,
                         _VP]),
    ("pals_replay_device", _I, [_VP, _I32, _VP, _VP, _VP, _VP, _VP, _I32, _VP, _I32, _VP, _VP,
                                _VP, _VP]),
    ("pals_replay_ex", _I, [_VP, _I32, _VP, _VP, _VP, _VP, _VP, _I32, _VP, _I32, _VP, _VP,
                            _VP, _VP, _VP]),
    ("pals_replay_device_ex", _I, [_VP, _I32, _VP, _VP, _VP, _VP, _VP, _I32, _VP, _I32, _VP,
                                   _VP, _VP, _VP, _VP]),
    ("pals_replay_traces", _I, [_VP, _I32, _VP, _VP, _VP, _VP, _VP, _I32, _VP, _I32, _VP,
                                _VP]),
    ("pals_replay_traces_device", _I, [_VP, _I32, _VP, _VP, _VP, _VP, _VP, _I32, _VP, _I32,
                                       _VP, _VP]),
    ("pals_replay_traces_status", _I64, [_VP]),
    ("pals_multi_create", _I, [_VP, _I32, _VP]),
    ("pals_multi_destroy", _I, [_VP]),
    ("pals_multi_size", _I32, [_VP]),
    ("pals_multi_ctx", _VP, [_VP, _I32]),
    ("pals_multi_set_gather", _I, [_VP, _I32]),
    ("pals_multi_model_analytic", _I, [_VP, _VP, _VP, _VP]),
    ("pals_multi_model_table", _I, [_VP, _VP, _VP, _VP, _I64, _VP]),
    ("pals_multi_select", _I, [_VP, _I32, _VP, _I64, _VP, _VP, _I64, _VP, _VP]),
    ("pals_multi_replay", _I, [_VP, _I32, _VP, _VP, _VP, _VP, _VP, _I32, _VP, _I32, _VP, _VP,
                               _VP, _VP, _VP]),
    ("pals_multi_replay_traces", _I, [_VP, _I32, _VP, _VP, _VP, _VP, _VP, _I32, _VP, _I32,
                                      _VP, _VP]),
    ("pals_multi_last_ms", _I, [_VP, _VP]),
    ("pals_decisions_csv", _I, [_VP, _VP, _I32, _VP, _I32, _VP, _I32, _VP, _VP, _VP, _VP, _I64,
                                _VP]),
    ("pals_fnv1a64", C.c_uint64, [_VP, _I64]),
    ("pals_sim_last_timing", _I, [_VP, _VP, _VP]),
    ("pals_sim_keep_requests", _I, [_VP, _I32]),
    ("pals_sim_set_streaming", _I, [_VP, _I32]),
    ("pals_sim_requests", _I, [_VP, _I64, _VP, _I64, _VP]),
    ("pals_run_scenarios", _I, [_VP, _I32, _VP, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _VP,
                                _VP]),
    ("pals_plan_frontier", _I, [_VP, _VP, _VP]),
    ("pals_plan_frontier_device", _I, [_VP, _VP, _VP]),
    ("pals_frontier_values", _I, [_VP, _VP, _VP, _VP, _I64, _VP, _VP]),
    ("pals_alloc_create", _I, [_VP, _I32, _VP, _VP, _VP, _VP, _VP, _I32, _VP, _I32, _I32, _D,
                               _VP]),
    ("pals_alloc_destroy", _I, [_VP]),
    ("pals_alloc_create_sets", _I, [_VP, _I32, _VP, _VP, _VP, _VP, _VP, _D, _VP]),
    ("pals_alloc_steps", _I, [_VP, _I32, _VP, _VP, _VP]),
    ("pals_allocate_budget", _I, [_VP, _D, _I64] + [_VP] * 9),
    ("pals_alloc_run_device", _I, [_VP, _D, _I64, _VP, _I64] + [_VP] * 8),
]

_lib = None


class PalsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[pals {code}] {msg}")
        self.code = code
        self.msg = msg


class ConfigError(PalsError):
    """wattserve::config_error (types.hpp:13-15)."""


class DataError(PalsError):
    """wattserve::data_error (types.hpp:17-19)."""


class OutOfRange(PalsError):
    """std::out_of_range (types.hpp:118-119, model.hpp:39-40)."""


_ERR = {abi.PALS_ECONFIG: ConfigError, abi.PALS_EDATA: DataError, abi.PALS_ERANGE: OutOfRange}


def load(build_if_missing: bool = True) -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise OSError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        from .build import build
        build()
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != abi.PALS_OK:
        msg = _lib.pals_last_error().decode(errors="replace")
        raise _ERR.get(rc, PalsError)(rc, msg)
