"""ctypes binding of librcseg_b200.so (include/rcb.h).

There is no CPU fallback: importing the product without the built library, or
calling a compute entry point on a machine without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RCB_LIB_PATH") or os.path.join(_HERE, "librcseg_b200.so")

RCB_OK = 0
RCB_ERR_VALUE = -1
RCB_ERR_CUDA = -2
RCB_ERR_CAPACITY = -3
RCB_ERR_DEGENERATE = -4
RCB_ERR_NODEVICE = -5


class EnergyCfg(C.Structure):
    _fields_ = [("region_model", C.c_int32), ("noise_model", C.c_int32), ("lam", C.c_double),
                ("smooth_radius", C.c_int32)]


class SobolevCfg(C.Structure):
    _fields_ = [("length_scale", C.c_double), ("epsilon", C.c_double),
                ("weights", C.POINTER(C.c_double)), ("n_weights", C.c_int32)]


class OptCfg(C.Structure):
    _fields_ = [("gradient", C.c_int32), ("move_budget", C.c_double), ("seed", C.c_uint64),
                ("allow_fusion", C.c_int32), ("allow_vanish", C.c_int32),
                ("vanish_grace", C.c_int32), ("full_fg", C.c_int32), ("fp32", C.c_int32)]


class SlabInfo(C.Structure):
    _fields_ = [("n_particles", C.c_int64), ("p0", C.c_int64), ("p1", C.c_int64),
                ("base", C.c_void_p), ("cb0", C.c_void_p), ("sb0", C.c_void_p),
                ("stream", C.c_void_p)]


class IterRecord(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("energy", C.c_double), ("moves", C.c_int64),
                ("particles", C.c_int64), ("candidates", C.c_int64), ("negative", C.c_int64),
                ("pairs", C.c_int64), ("mode", C.c_int32)]


_P = C.c_void_p
_I32, _I64, _D = C.c_int32, C.c_int64, C.c_double

# name -> argtypes (all return int32 status unless listed in _VOID)
SIGNATURES = {
    "rcb_version": [],
    "rcb_last_error": [],
    "rcb_device_count": [_P],
    "rcb_sobolev_filter": [_P, _I64, _I32, _P, _P, _P, _P, _P, _P],
    "rcb_scan_contour": [_P, _I32, _P, _I32, _P, _P, _P, _I64, _P],
    "rcb_delta_internal_batch": [_P, _I32, _P, _P, _P, _P, _I64, _P],
    "rcb_delta_external_batch": [_P, _P, _I32, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _I64, _P],
    "rcb_stats_from_labels": [_P, _P, _I64, _I32, _P, _P, _P],
    "rcb_evaluate_total": [_P, _P, _I32, _P, _P, _P, _P],
    "rcb_label_components": [_P, _I32, _P, _I32, _I32, _I64, _P, _P],
    "rcb_moves_admissible": [_P, _I32, _P, _I32, _P, _P, _P, _I64, _I32, _I32, _P],
    "rcb_cell_pairs": [_P, _I64, _I32, _D, _D, _P, _P, _P, _I64, _P],
    "rcb_cell_query": [_P, _I64, _I32, _D, _P, _D, _I64, _P, _P],
    "rcb_ball_sum": [_P, _I32, _P, _I32, _P],
    "rcb_smooth_fields": [_P, _P, _I32, _P, _I32, _I32, _P, _P],
    "rcb_engine_create": [_P, _P, _I32, _P, _P, _P, _P, _I32, _P, _P],
    "rcb_engine_create_ex": [_P, _I32, _P, _I32, _P, _P, _P, _P, _I32, _P, _P],
    "rcb_engine_destroy": [_P],
    "rcb_engine_iterate": [_P, _P],
    "rcb_engine_get_labels": [_P, _P],
    "rcb_engine_set_labels": [_P, _P],
    "rcb_engine_undo_last": [_P],
    "rcb_engine_get_candidates": [_P, _P, _P, _P, _P, _I64, _P],
    "rcb_engine_get_accepted": [_P, _P, _I64, _P],
    "rcb_engine_get_stats": [_P, _P, _P, _P, _I32],
    "rcb_engine_n_labels": [_P, _P],
    "rcb_engine_set_mode": [_P, _I32],
    "rcb_engine_set_energy": [_P, _D],
    "rcb_engine_refresh": [_P],
    "rcb_engine_evaluate": [_P, _P, _P],
    "rcb_engine_stream": [_P, _P],
    "rcb_engine_timings": [_P, _P, _P],
    "rcb_engine_counters": [_P, _P],
    "rcb_engine_debug_codes": [_P, _P, _P, _I64, _P],
    "rcb_engine_debug_times": [_P, _P, _I64, _P],
    "rcb_engine_set_slab": [_P, _I64, _I64],
    "rcb_engine_score": [_P, _P],
    "rcb_engine_finish": [_P, _P],
    "rcb_engine_band_limbs": [_P, _P, _P, _P, _P],
    "rcb_engine_band_apply": [_P, _P],
    "rcb_engine_particle_ranges": [_P, _P, _I32, _P],
    "rcb_synth_generate": [_I32, _P, _D, _P, _I32, _P, _I32, _I32, _D, C.c_uint64, _P, _P, _P],
    "rcb_synth_blur": [_P, _I32, _P, _P, _I32, _P],
    "rcb_synth_poissonize": [_P, _I64, _D, C.c_uint64, _P],
    "rcb_sweep_create": [_I32, _P, _P, _I32, C.c_uint64, _P, _I32, _P],
    "rcb_sweep_destroy": [_P],
    "rcb_sweep_info": [_P, _P, _P, _P],
    "rcb_sweep_run": [_P, _P, _P],
    "rcb_sweep_get": [_P, _P, _P, _P, _P, _P, _I64],
}
_RESTYPES = {"rcb_last_error": C.c_char_p, "rcb_engine_destroy": None, "rcb_sweep_destroy": None}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built: run `make` (or __graft_entry__.build()) — "
            "there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, C.c_int32)
    return lib


lib = _load()


class DegenerateStatsError(RuntimeError):
    """A required region mean is undefined (energy.py:33-34)."""


def check(status: int) -> None:
    if status == RCB_OK:
        return
    msg = (lib.rcb_last_error() or b"").decode(errors="replace")
    if status == RCB_ERR_VALUE:
        raise ValueError(msg)
    if status == RCB_ERR_DEGENERATE:
        raise DegenerateStatsError(msg)
    raise RuntimeError(f"librcseg_b200 status {status}: {msg}")


def device_count() -> int:
    n = C.c_int32(0)
    lib.rcb_device_count(C.byref(n))
    return n.value


def require_device() -> None:
    if device_count() < 1:
        raise RuntimeError("librcseg_b200 needs a CUDA device (B200); there is no CPU fallback")


def ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def c64(a, dtype=np.int64) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def dims_arr(shape) -> np.ndarray:
    return np.ascontiguousarray(np.array(shape, dtype=np.int64))
