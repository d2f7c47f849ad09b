"""ctypes binding of libevsim_b200.so (the C ABI in include/evsim_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libevsim_b200.so")

EVS_OK = 0
EVS_ERR_ARG = 1
EVS_ERR_CUDA = 2
EVS_ERR_WORKSPACE = 3
EVS_ERR_UNSUPPORTED = 4
EVS_ORDER_PIXEL_MAJOR = 0
EVS_ORDER_CANONICAL = 1
EVS_EPOCHS_PER_CALL = 8
EVS_EPOCH_LIMIT = (1 << 22) - 1
NO_BAD = 0x7FFFFFFFFFFFFFFF

# Every symbol include/evsim_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTED_SYMBOLS = (
    "evs_version", "evs_error_string", "evs_step_workspace_bytes", "evs_step",
    "evs_step_profiled", "evs_step_clock_init",
    "evs_sort_workspace_bytes", "evs_canonical_sort", "evs_sort_general_workspace_bytes",
    "evs_canonical_sort_general", "evs_batch_stats", "evs_seed_pcg64",
    "evs_noise_workspace_bytes", "evs_noise", "evs_noise_batch_workspace_bytes", "evs_noise_batch",
    "evs_accumulate", "evs_voxel", "evs_voxel_segments", "evs_step_voxel", "evs_step_histogram",
    "evs_compact_segments", "evs_pack_segments", "evs_merge_runs", "evs_log_transform",
    "evs_limit_bandwidth_workspace_bytes", "evs_limit_bandwidth", "evs_render",
)


class StepParams(ctypes.Structure):
    _fields_ = [
        ("streams", ctypes.c_int32), ("frames", ctypes.c_int32),
        ("height", ctypes.c_int32), ("width", ctypes.c_int32),
        ("log_eps", ctypes.c_double), ("refractory_us", ctypes.c_int64),
        ("capacity", ctypes.c_int64),
        ("th_pos_uniform", ctypes.c_float), ("th_neg_uniform", ctypes.c_float),
        ("t0", ctypes.c_int64), ("tick", ctypes.c_int64), ("max_dt", ctypes.c_int64),
        ("order", ctypes.c_int32), ("validate", ctypes.c_int32),
        ("epoch", ctypes.c_uint32), ("flags", ctypes.c_int32), ("clock_stride", ctypes.c_int32),
        ("keys_hint", ctypes.c_int64),
    ]


EVS_FLAG_DEVICE_CLOCK = 1


class RenderPlane(ctypes.Structure):  # evs_plane
    _fields_ = [("axis", ctypes.c_int32), ("kind", ctypes.c_int32), ("offset", ctypes.c_double),
                ("bounds", ctypes.c_double * 4), ("cell", ctypes.c_double), ("value_a", ctypes.c_double),
                ("value_b", ctypes.c_double), ("seed", ctypes.c_uint64)]


class RenderParams(ctypes.Structure):  # evs_render_params
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("rot", ctypes.c_double * 9), ("origin", ctypes.c_double * 3), ("ambient", ctypes.c_double)]


EVS_TEX_CHECKER = 0
EVS_TEX_NOISE = 1
EVS_VOXEL_CLEAR = 1
EVS_VOXEL_FINALIZE = 2


class StepBuffers(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "frames", "t_bounds", "ref_log", "last_event_t", "th_pos", "th_neg",
        "ev_t", "ev_x", "ev_y", "ev_p", "counts", "dropped", "reservations", "bad_pixel")]


class NoiseParams(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32), ("height", ctypes.c_int32),
        ("t_prev", ctypes.c_int64), ("t_now", ctypes.c_int64),
        ("lam", ctypes.c_double), ("enlam", ctypes.c_double),
        ("pcg", ctypes.c_uint64 * 4),
        ("capacity", ctypes.c_int64), ("order", ctypes.c_int32), ("reserved", ctypes.c_uint32),
        ("draw_scale", ctypes.c_double),
    ]


_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    pass


def load():
    """Load (building if needed) the native library; raise if impossible."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            from . import build as _b
            _b.build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        u32 = ctypes.c_uint32
        sz = ctypes.c_size_t
        L.evs_version.restype = ctypes.c_int
        L.evs_error_string.restype = ctypes.c_char_p
        L.evs_error_string.argtypes = [ctypes.c_int]
        L.evs_step_workspace_bytes.restype = sz
        L.evs_step_workspace_bytes.argtypes = [ctypes.POINTER(StepParams)]
        L.evs_step.argtypes = [ctypes.POINTER(StepParams), ctypes.POINTER(StepBuffers), P, sz, P]
        L.evs_step_profiled.argtypes = [ctypes.POINTER(StepParams), ctypes.POINTER(StepBuffers), P, sz,
                                        P, P, ctypes.c_int32]
        L.evs_step_clock_init.argtypes = [ctypes.POINTER(StepParams), P, sz, i64, u32, P]
        L.evs_sort_workspace_bytes.restype = sz
        L.evs_sort_workspace_bytes.argtypes = [i64, i64]
        L.evs_canonical_sort.argtypes = [i64, P, P, P, P, i64, i64, u32, P, sz, P]
        L.evs_sort_general_workspace_bytes.restype = sz
        L.evs_sort_general_workspace_bytes.argtypes = [i64]
        L.evs_canonical_sort_general.argtypes = [i64, P, P, P, P, P, sz, P]
        L.evs_batch_stats.argtypes = [i64, P, P, P, P, P, P]
        L.evs_seed_pcg64.argtypes = [P, ctypes.c_int32, P]
        L.evs_seed_pcg64.restype = None
        _bind_extras(L)
        _lib = L
        return L


def _bind_extras(L) -> None:
    """argtypes of the representation / noise entry points."""
    P = ctypes.c_void_p
    i64 = ctypes.c_int64
    i32 = ctypes.c_int32
    sz = ctypes.c_size_t
    L.evs_noise_workspace_bytes.restype = sz
    L.evs_noise_workspace_bytes.argtypes = [ctypes.POINTER(NoiseParams)]
    L.evs_noise_capacity.restype = i64
    L.evs_noise_capacity.argtypes = [ctypes.POINTER(NoiseParams)]
    L.evs_noise.argtypes = [ctypes.POINTER(NoiseParams), P, P, P, P, P, P, P, sz, P]
    L.evs_noise_batch_workspace_bytes.restype = sz
    L.evs_noise_batch_workspace_bytes.argtypes = [P, i32]
    L.evs_noise_batch.argtypes = [P, i32, P, P, P, P, i64, P, P, sz, P]
    L.evs_accumulate.argtypes = [i64, P, P, P, P, i64, i64, i32, i32, P, P]
    L.evs_voxel_workspace_bytes.restype = sz
    L.evs_voxel_workspace_bytes.argtypes = [i32, i32, i32]
    L.evs_voxel.argtypes = [i64, P, P, P, P, i64, i64, i32, i32, i32, P, P, sz, P]
    L.evs_voxel_segments.argtypes = [i32, P, i64, i64, P, P, P, P, i64, i64, i32, i32, i32, i32, P, P, sz, P]
    L.evs_step_voxel.argtypes = [P, P, P, sz, i32, i64, i64, i32, i32, P, P, sz, P]
    L.evs_step_histogram.argtypes = [P, P, P, sz, i64, i64, P, P]
    L.evs_compact_segments.argtypes = [i32, P, i64, P, P, P, P, P, P, P, P, i64, P]
    L.evs_pack_segments.argtypes = [i32, P, i64, P, P, P, P, i64, i32, i32, i32, i32, P, P, i64, P]
    L.evs_merge_runs.argtypes = [i32, P, i64, P, P, P]
    L.evs_log_transform.argtypes = [i64, P, ctypes.c_double, P, P, P]
    L.evs_limit_bandwidth_workspace_bytes.restype = sz
    L.evs_limit_bandwidth_workspace_bytes.argtypes = [i64]
    L.evs_limit_bandwidth.argtypes = [i64, P, P, P, P, i64, i64, P, P, P, P, P, P, sz, P]
    L.evs_selftest_log.argtypes = [i64, P, P, P, P]
    L.evs_merge_canonical.argtypes = [i64, P, P, P, P, i64, P, P, P, P, i64, P, P, P, P, P, sz, P]
    L.evs_render.argtypes = [ctypes.POINTER(RenderParams), P, i32, P, P, P]


def check(rc: int, what: str) -> None:
    if rc != EVS_OK:
        msg = load().evs_error_string(rc).decode()
        if rc in (EVS_ERR_ARG,):
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what}: {msg} (status {rc})")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeError("paper_2602_15018_b200 requires a CUDA device (B200, sm_100a); "
                          "there is no CPU fallback")
    load()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class EpochCounter:
    """Caller-side epoch management for a workspace (see EVS_EPOCHS_PER_CALL)."""

    def __init__(self):
        self.value = 1

    def take(self, workspace) -> int:
        if self.value + EVS_EPOCHS_PER_CALL > EVS_EPOCH_LIMIT:
            workspace.zero_()
            self.value = 1
        e = self.value
        self.value += EVS_EPOCHS_PER_CALL
        return e
