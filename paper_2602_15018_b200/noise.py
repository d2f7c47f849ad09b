"""Exact background noise (inject_noise_events, model.py:174-212) on the GPU.

The host does only what numpy does on the host side of the reference: it
derives lam = rate * (dt * 1e-6), exp(-lam) (libm) and the PCG64 state of
``default_rng(seed)`` (SeedSequence, ported in evs_seed_pcg64); the draws,
Poisson counts, timestamps, polarities and the per-pixel ordering run in the
noise kernels (csrc/noise.cu).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .events.types import DeviceEventBatch, EventBatch

_ws_cache: dict = {}


def seed_words(seed: int) -> np.ndarray:
    """numpy _coerce_to_uint32_array for a non-negative integer seed (LSW first)."""
    seed = int(seed)
    if seed < 0:
        raise ValueError("expected non-negative integer")
    words = []
    while True:
        words.append(seed & 0xFFFFFFFF)
        seed >>= 32
        if seed == 0:
            break
    return np.array(words, np.uint32)


def pcg64_state(seed: int) -> np.ndarray:
    """(state_hi, state_lo, inc_hi, inc_lo) of numpy default_rng(seed), via the C ABI."""
    w = seed_words(seed)
    out = np.zeros(4, np.uint64)
    _lib.load().evs_seed_pcg64(w.ctypes.data, len(w), out.ctypes.data)
    return out


def noise_params(width, height, t_prev, t_now, noise_rate_hz, seed, order=0) -> _lib.NoiseParams:
    dt_us = int(t_now) - int(t_prev)
    lam = noise_rate_hz * (dt_us * 1e-6)  # model.py:195 (same float operations)
    p = _lib.NoiseParams()
    p.width, p.height = int(width), int(height)
    p.t_prev, p.t_now = int(t_prev), int(t_now)
    p.lam = lam
    p.enlam = math.exp(-lam)
    st = pcg64_state(seed)
    for i in range(4):
        p.pcg[i] = int(st[i])
    p.capacity = 0
    p.order = order
    p.draw_scale = 1.0
    return p


def run_noise(p: _lib.NoiseParams, device, stream=None):
    """Launch evs_noise with retries; returns (count, buffers) on `device`."""
    import torch

    L = _lib.load()
    for _attempt in range(8):
        cap = int(L.evs_noise_capacity(ctypes.byref(p)))
        nbytes = int(L.evs_noise_workspace_bytes(ctypes.byref(p)))
        key = (device, "noise")
        ws = _ws_cache.get(key)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
            _ws_cache[key] = ws
        meta = torch.zeros(4, dtype=torch.int64, device=device)
        if p.order == 1:
            bufs = {"key": torch.empty(cap, dtype=torch.int64, device=device)}
            ptrs = (None, None, None, None, bufs["key"].data_ptr())
        else:
            bufs = {"t": torch.empty(cap, dtype=torch.int64, device=device),
                    "x": torch.empty(cap, dtype=torch.int16, device=device),
                    "y": torch.empty(cap, dtype=torch.int16, device=device),
                    "p": torch.empty(cap, dtype=torch.int8, device=device)}
            ptrs = (bufs["t"].data_ptr(), bufs["x"].data_ptr(), bufs["y"].data_ptr(), bufs["p"].data_ptr(), None)
        rc = L.evs_noise(ctypes.byref(p), *ptrs, meta.data_ptr(), ws.data_ptr(), ws.numel(),
                         _lib.stream_ptr(stream))
        _lib.check(rc, "evs_noise")
        m = meta.cpu().tolist()
        if m[2]:
            p.draw_scale = max(2.0, p.draw_scale * 2.0)
            continue
        if m[3]:
            p.capacity = int(m[1]) + 1024
            continue
        return int(m[1]), bufs
    raise _lib.NativeError("evs_noise did not converge (draw range / capacity retries exhausted)")


def noise_events(width: int, height: int, t_prev: int, t_now: int, noise_rate_hz: float, seed: int,
                 device_output: bool = False):
    """inject_noise_events (model.py:174-212); host EventBatch unless device_output."""
    if noise_rate_hz < 0:
        raise ValueError("noise_rate_hz must be >= 0")
    if t_now <= t_prev:
        raise ValueError(f"t_now ({t_now}) must be greater than t_prev ({t_prev})")
    if noise_rate_hz == 0:
        return EventBatch.empty()
    _lib.require_cuda()
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    p = noise_params(width, height, t_prev, t_now, noise_rate_hz, seed)
    if p.lam <= 0:
        return EventBatch.empty()
    n, b = run_noise(p, dev)
    if n == 0:
        return EventBatch.empty()
    db = DeviceEventBatch(b["t"][:n], b["x"][:n], b["y"][:n], b["p"][:n], 0, False)
    return db if device_output else db.to_host()
