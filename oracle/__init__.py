"""CPU oracle for the event-camera hot path -- TEST INFRASTRUCTURE ONLY.

This package restates the reference's algorithm (``evsim.events``,
/root/reference/pkg/src/evsim/events) in plain C (``evsim_oracle.c``) with a
thin numpy/ctypes wrapper.  It is the parity checker: only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The product package
(``paper_2602_15018_b200``) never imports it and has no CPU fallback.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``).

The log front-end (model.py:28-39) is computed here with numpy exactly as the
reference does (``np.log(values.astype(float64) + log_eps)``) and handed to
the C lane math, so the oracle shares the reference's log on any host.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")
_lib = None

CROSSING_TOL = 1e-4  # types.py:22
MIN_THRESHOLD = 0.01  # types.py:17
CHUNK_WIDTH = 32  # parallel.py:32


def build(force: bool = False) -> str:
    """Compile liborc.so with the committed Makefile (gcc)."""
    src = os.path.join(_HERE, "evsim_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liborc.so"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        d = ctypes.c_double
        L.orc_generate_serial.argtypes = [i64, i64, P, P, P, P, P, P, i64, i64, d, i64, i64, i64,
                                          P, P, P, P, P, P, P, P]
        L.orc_generate_mt.argtypes = [i64, i64, P, P, P, P, P, i64, i64, d, i64, i64, i64,
                                      P, P, P, P, P, P, P, P, ctypes.c_int]
        L.orc_canonical_sort.argtypes = [i64, P, P, P, P]
        L.orc_accumulate.argtypes = [i64, P, P, P, P, i64, i64, i64, i64, P]
        L.orc_voxel.argtypes = [i64, P, P, P, P, i64, i64, i64, i64, i64, P]
        L.orc_limit_bandwidth.argtypes = [i64, P, d, i64, P, P]
        L.orc_seed_pcg64.argtypes = [P, ctypes.c_int, P]
        L.orc_seed_pcg64.restype = None
        L.orc_noise.argtypes = [i64, i64, i64, i64, d, P, i64, P, P, P, P, P]
        L.orc_pcg64_draws.argtypes = [P, i64, P]
        L.orc_pcg64_draws.restype = None
        L.orc_first_bad_pixel.argtypes = [i64, P]
        L.orc_first_bad_pixel.restype = i64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class OBatch:
    """Oracle event batch: same SoA layout and dtypes as evsim EventBatch (types.py:34-42)."""

    t: np.ndarray  # uint64
    x: np.ndarray  # uint16
    y: np.ndarray  # uint16
    polarity: np.ndarray  # int8
    dropped_count: int = 0
    reservation_count: int = 0

    def __len__(self) -> int:
        return len(self.t)

    def same_events(self, other) -> bool:
        """types.py:71-79, order-sensitive equality."""
        return (len(self) == len(other)
                and np.array_equal(np.asarray(self.t, np.uint64), np.asarray(other.t, np.uint64))
                and np.array_equal(np.asarray(self.x), np.asarray(other.x))
                and np.array_equal(np.asarray(self.y), np.asarray(other.y))
                and np.array_equal(np.asarray(self.polarity), np.asarray(other.polarity)))


@dataclass
class OState:
    """PixelStateGrid restatement (types.py:159-178)."""

    width: int
    height: int
    ref_log: np.ndarray  # float32 (h, w)
    last_event_t: np.ndarray  # int64 (h, w)
    thresholds_pos: np.ndarray  # float32 (h, w)
    thresholds_neg: np.ndarray  # float32 (h, w)

    def copy(self) -> "OState":
        return OState(self.width, self.height, self.ref_log.copy(), self.last_event_t.copy(),
                      self.thresholds_pos.copy(), self.thresholds_neg.copy())


def log_transform(values: np.ndarray, log_eps: float) -> np.ndarray:
    """model.py:28-39."""
    if log_eps <= 0:
        raise ValueError("log_eps must be positive")
    vals = np.asarray(values, np.float32)
    bad = ~np.isfinite(vals) | (vals < 0.0) | (vals > 1.0)
    if bad.any():
        yy, xx = np.nonzero(bad)
        raise ValueError(f"invalid intensity {vals[yy[0], xx[0]]!r} at pixel (x={xx[0]}, y={yy[0]})")
    return np.log(vals.astype(np.float64) + log_eps)


def init_state(frame0: np.ndarray, c_pos=0.2, c_neg=0.2, sigma_c=0.0, refractory_us=0,
               log_eps=0.01, seed=0, t0=0) -> OState:
    """init_pixel_states, model.py:42-67 (threshold normals drawn with numpy, as the reference)."""
    h, w = frame0.shape
    ref = log_transform(frame0, log_eps).astype(np.float32)
    rng = np.random.default_rng(seed)
    if sigma_c > 0:
        thp = rng.normal(c_pos, sigma_c, size=(h, w))
        thn = rng.normal(c_neg, sigma_c, size=(h, w))
    else:
        thp = np.full((h, w), c_pos)
        thn = np.full((h, w), c_neg)
    thp = np.maximum(thp, MIN_THRESHOLD).astype(np.float32)
    thn = np.maximum(thn, MIN_THRESHOLD).astype(np.float32)
    last = np.full((h, w), int(t0) - int(refractory_us), np.int64)
    return OState(w, h, ref, last, thp, thn)


def generate(state: OState, frame: np.ndarray, t_prev: int, t_now: int, log_eps=0.01,
             refractory_us=0, cap=None, nthreads: int = 0) -> OBatch:
    """generate_events_serial (model.py:79-171): pixel-major order, mutates state.

    nthreads > 0 uses the banded multithreaded C port (identical output) with
    the C library log -- used only as the CPU baseline.
    """
    L = lib()
    frame = np.ascontiguousarray(frame, np.float32)
    h, w = state.height, state.width
    if frame.shape != (h, w):
        raise ValueError(f"frame {frame.shape[1]}x{frame.shape[0]} does not match state {w}x{h}")
    if t_now <= t_prev:
        raise ValueError(f"t_now ({t_now}) must be greater than t_prev ({t_prev})")
    if cap is None:
        cap = 8 * w * h
    lnew = None
    if nthreads <= 0:
        lnew = log_transform(frame, log_eps)  # raises like the reference
    n_guess = min(cap, max(16, 3 * w * h))
    for _attempt in range(3):
        out_t = np.empty(n_guess, np.int64)
        out_x = np.empty(n_guess, np.uint16)
        out_y = np.empty(n_guess, np.uint16)
        out_p = np.empty(n_guess, np.int8)
        n = np.zeros(1, np.int64)
        dropped = np.zeros(1, np.int64)
        res = np.zeros(1, np.int64)
        bad = np.zeros(1, np.int64)
        ref_bak = state.ref_log.copy()
        last_bak = state.last_event_t.copy()
        args = [h, w, _p(frame)]
        if nthreads <= 0:
            args.append(_p(lnew))
            fn = L.orc_generate_serial
        else:
            fn = L.orc_generate_mt
        args += [_p(state.ref_log), _p(state.last_event_t), _p(state.thresholds_pos),
                 _p(state.thresholds_neg), int(t_prev), int(t_now), float(log_eps),
                 int(refractory_us), int(cap), n_guess, _p(out_t), _p(out_x), _p(out_y),
                 _p(out_p), _p(n), _p(dropped), _p(res), _p(bad)]
        if nthreads > 0:
            args.append(int(nthreads))
        rc = fn(*args)
        if rc == 1:
            b = int(bad[0])
            yy, xx = divmod(b, w)
            raise ValueError(f"invalid intensity {frame[yy, xx]!r} at pixel (x={xx}, y={yy})")
        if rc == 4:  # output too small: restore and retry bigger
            state.ref_log[...] = ref_bak
            state.last_event_t[...] = last_bak
            n_guess = min(cap, n_guess * 4) if n_guess < cap else cap
            continue
        if rc != 0:
            raise RuntimeError(f"oracle rc={rc}")
        k = int(n[0])
        return OBatch(out_t[:k].astype(np.uint64), out_x[:k].copy(), out_y[:k].copy(),
                      out_p[:k].copy(), int(dropped[0]), int(res[0]))
    raise RuntimeError("oracle output sizing failed")


def canonical_sort(b: OBatch) -> OBatch:
    """parallel.py:112-123."""
    t = np.asarray(b.t).astype(np.int64).copy()
    x = np.asarray(b.x, np.uint16).copy()
    y = np.asarray(b.y, np.uint16).copy()
    p = np.asarray(b.polarity, np.int8).copy()
    rc = lib().orc_canonical_sort(len(t), _p(t), _p(x), _p(y), _p(p))
    assert rc == 0
    return OBatch(t.astype(np.uint64), x, y, p, b.dropped_count, b.reservation_count)


def concat(batches) -> OBatch:
    """types.py:82-92."""
    if not batches:
        return OBatch(np.empty(0, np.uint64), np.empty(0, np.uint16), np.empty(0, np.uint16),
                      np.empty(0, np.int8))
    return OBatch(np.concatenate([np.asarray(b.t, np.uint64) for b in batches]),
                  np.concatenate([np.asarray(b.x, np.uint16) for b in batches]),
                  np.concatenate([np.asarray(b.y, np.uint16) for b in batches]),
                  np.concatenate([np.asarray(b.polarity, np.int8) for b in batches]),
                  sum(b.dropped_count for b in batches))


def accumulate(b, window_us: int, t_end: int, width: int, height: int) -> np.ndarray:
    """accumulate_events_to_image, model.py:249-262."""
    t = np.ascontiguousarray(np.asarray(b.t).astype(np.int64))
    x = np.ascontiguousarray(b.x, np.uint16)
    y = np.ascontiguousarray(b.y, np.uint16)
    p = np.ascontiguousarray(b.polarity, np.int8)
    g = np.zeros((height, width), np.int64)
    rc = lib().orc_accumulate(len(t), _p(t), _p(x), _p(y), _p(p), int(window_us), int(t_end),
                              int(width), int(height), _p(g))
    if rc != 0:
        raise ValueError("event coordinates out of bounds for the given dimensions")
    return g


def voxel(b, t0: int, t1: int, bins: int, width: int, height: int) -> np.ndarray:
    """Voxel grid (repo-defined): exact integer bilinear-in-time weights."""
    t = np.ascontiguousarray(np.asarray(b.t).astype(np.int64))
    x = np.ascontiguousarray(b.x, np.uint16)
    y = np.ascontiguousarray(b.y, np.uint16)
    p = np.ascontiguousarray(b.polarity, np.int8)
    v = np.zeros((bins, height, width), np.float32)
    rc = lib().orc_voxel(len(t), _p(t), _p(x), _p(y), _p(p), int(t0), int(t1), int(bins),
                         int(width), int(height), _p(v))
    if rc != 0:
        raise ValueError("bad voxel arguments")
    return v


def limit_bandwidth(b, max_events_per_sec: float, window_us: int) -> OBatch:
    """model.py:215-246."""
    if window_us <= 0:
        raise ValueError("window_us must be positive")
    if max_events_per_sec < 0:
        raise ValueError("max_events_per_sec must be >= 0")
    t = np.ascontiguousarray(np.asarray(b.t).astype(np.int64))
    keep = np.zeros(len(t), np.uint8)
    nd = np.zeros(1, np.int64)
    if len(t) == 0:
        return OBatch(t.astype(np.uint64), np.asarray(b.x), np.asarray(b.y),
                      np.asarray(b.polarity), b.dropped_count)
    rc = lib().orc_limit_bandwidth(len(t), _p(t), float(max_events_per_sec), int(window_us),
                                   _p(keep), _p(nd))
    if rc != 0:
        raise ValueError("limit_bandwidth requires a timestamp-sorted batch")
    k = keep.astype(bool)
    return OBatch(np.asarray(b.t, np.uint64)[k], np.asarray(b.x)[k], np.asarray(b.y)[k],
                  np.asarray(b.polarity)[k], b.dropped_count + int(nd[0]))


def mix64(*parts: int) -> int:
    """orchestrator.py:51-56 (FNV-style seed mixing)."""
    h = 0xCBF29CE484222325
    for p in parts:
        h ^= p & 0xFFFFFFFFFFFFFFFF
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def seed_words(seed: int) -> np.ndarray:
    """numpy _coerce_to_uint32_array for a non-negative int seed (LSW first)."""
    seed = int(seed)
    if seed < 0:
        raise ValueError("seed must be non-negative")
    words = []
    while True:
        words.append(seed & 0xFFFFFFFF)
        seed >>= 32
        if seed == 0:
            break
    return np.array(words, np.uint32)


def pcg64_state(seed: int) -> np.ndarray:
    """default_rng(seed) PCG64 (state_hi, state_lo, inc_hi, inc_lo)."""
    w = seed_words(seed)
    out = np.zeros(4, np.uint64)
    lib().orc_seed_pcg64(_p(w), len(w), _p(out))
    return out


def pcg64_draws(seed: int, n: int) -> np.ndarray:
    st = pcg64_state(seed)
    out = np.zeros(n, np.uint64)
    lib().orc_pcg64_draws(_p(st), int(n), _p(out))
    return out


def noise(width: int, height: int, t_prev: int, t_now: int, rate: float, seed: int) -> OBatch:
    """inject_noise_events, model.py:174-212 (exact numpy draw order)."""
    if rate < 0:
        raise ValueError("noise_rate_hz must be >= 0")
    if t_now <= t_prev:
        raise ValueError(f"t_now ({t_now}) must be greater than t_prev ({t_prev})")
    st = pcg64_state(seed)
    cap = 1024
    while True:
        out_t = np.empty(cap, np.int64)
        out_x = np.empty(cap, np.uint16)
        out_y = np.empty(cap, np.uint16)
        out_p = np.empty(cap, np.int8)
        n = np.zeros(1, np.int64)
        rc = lib().orc_noise(int(width), int(height), int(t_prev), int(t_now), float(rate),
                             _p(st), cap, _p(out_t), _p(out_x), _p(out_y), _p(out_p), _p(n))
        if rc == 4:
            cap = int(n[0])
            continue
        if rc != 0:
            raise RuntimeError(f"oracle noise rc={rc}")
        k = int(n[0])
        return OBatch(out_t[:k].astype(np.uint64), out_x[:k].copy(), out_y[:k].copy(),
                      out_p[:k].copy())


def texture_frame(width: int, height: int, phase: float) -> np.ndarray:
    """_texture_frame, events_bench.py:19-26 (f64 math, cast to f32)."""
    x = np.arange(width) / width
    y = np.arange(height) / height
    grid = np.add.outer(y * 2.0, x * 3.0)
    return (0.5 + 0.45 * np.sin(2.0 * np.pi * (grid + phase))).astype(np.float32)


def frame_from_log(log_vals, log_eps: float = 0.01) -> np.ndarray:
    """helpers.py:10-16."""
    vals = np.exp(np.asarray(log_vals, np.float64)) - log_eps
    return np.clip(vals, 0.0, 1.0).astype(np.float32)


def random_walk_sequence(rng, width, height, frames, step_std=0.08, lo=-4.0, hi=-0.1):
    """helpers.py:33-49 (values only; frame k is at t = k * tick)."""
    L = rng.uniform(lo + 1.0, hi - 1.0, (height, width))
    out = [frame_from_log(L)]
    for _k in range(1, frames):
        L = np.clip(L + rng.normal(0.0, step_std, (height, width)), lo, hi)
        out.append(frame_from_log(L))
    return out
