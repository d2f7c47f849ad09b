"""Contrast-threshold event generation: drop-in mirror of ``evsim.events.model``.

Reference: /root/reference/pkg/src/evsim/events/model.py.  The per-frame
work runs in the sm_100a kernels of ``libevsim_b200.so`` through the C ABI
(``evs_step``); there is no CPU fallback.  Host code here only validates
arguments, moves frames in and events out, and raises the reference's errors.
"""

from __future__ import annotations

import numpy as np

from .. import _lib
from ..runtime import PinnedPool, StepEngine, StepShape, d2h_rows, upload_frame
from .types import (
    MIN_THRESHOLD,
    DeviceEventBatch,
    EventBatch,
    EventCameraConfig,
    IntensityFrame,
    PixelStateGrid,
    _is_torch,
)


def _host_values(frame: IntensityFrame) -> np.ndarray:
    v = frame.values
    return v.detach().cpu().numpy() if _is_torch(v) else v


def _bad_pixel_error(values, flat: int, width: int) -> ValueError:
    yy, xx = divmod(int(flat), width)
    if _is_torch(values):
        val = np.float32(values.reshape(-1)[int(flat)].item())
    else:
        val = values[yy, xx]
    return ValueError(f"invalid intensity {val!r} at pixel (x={xx}, y={yy})")


def log_transform(frame: IntensityFrame, log_eps: float) -> np.ndarray:
    """model.py:28-39: per-pixel ln(I + log_eps) in float64; validates the frame.

    One pass of the evs_log_transform kernel (f64 log, <= 1 ulp; the first
    invalid pixel by atomicMin); returned as a host array like the reference.
    """
    import torch

    if log_eps <= 0:
        raise ValueError("log_eps must be positive")
    _lib.require_cuda()
    v = frame.values
    d = (v if _is_torch(v) else torch.from_numpy(np.ascontiguousarray(v, np.float32))).cuda()
    d = d.to(torch.float32).contiguous()
    out = torch.empty(d.shape, dtype=torch.float64, device=d.device)
    bad = torch.full((1,), _lib.NO_BAD, dtype=torch.int64, device=d.device)
    rc = _lib.load().evs_log_transform(d.numel(), d.data_ptr(), float(log_eps), out.data_ptr(), bad.data_ptr(),
                                       _lib.stream_ptr())
    _lib.check(rc, "evs_log_transform")
    flat = int(bad.item())
    if flat != _lib.NO_BAD:
        raise _bad_pixel_error(v, flat, frame.width)
    return out.cpu().numpy()


def init_pixel_states(frame0: IntensityFrame, config: EventCameraConfig, seed: int) -> PixelStateGrid:
    """model.py:42-67.

    One-time constructor work (reference level, threshold jitter) is done on
    the host with numpy so the thresholds are the reference's exact ziggurat
    normals for the seed; the grid is then uploaded and stays in HBM.
    """
    h, w = frame0.height, frame0.width
    vals = _host_values(frame0).astype(np.float32, copy=False)
    if config.log_eps <= 0:
        raise ValueError("log_eps must be positive")
    bad = ~np.isfinite(vals) | (vals < 0.0) | (vals > 1.0)
    if bad.any():
        yy, xx = np.nonzero(bad)
        raise ValueError(f"invalid intensity {vals[yy[0], xx[0]]!r} at pixel (x={xx[0]}, y={yy[0]})")
    ref = np.log(vals.astype(np.float64) + config.log_eps).astype(np.float32)
    rng = np.random.default_rng(seed)
    if config.sigma_c > 0:
        thp = rng.normal(config.c_pos, config.sigma_c, size=(h, w))
        thn = rng.normal(config.c_neg, config.sigma_c, size=(h, w))
    else:
        thp = np.full((h, w), config.c_pos)
        thn = np.full((h, w), config.c_neg)
    thp = np.maximum(thp, MIN_THRESHOLD).astype(np.float32)
    thn = np.maximum(thn, MIN_THRESHOLD).astype(np.float32)
    last_t = np.full((h, w), int(frame0.t) - int(config.refractory_us), np.int64)
    return PixelStateGrid(width=w, height=h, ref_log=ref, last_event_t=last_t,
                          thresholds_pos=thp, thresholds_neg=thn)


def _check_step(state: PixelStateGrid, frame: IntensityFrame, t_prev: int, t_now: int) -> None:
    """model.py:70-76."""
    if frame.width != state.width or frame.height != state.height:
        raise ValueError(
            f"frame {frame.width}x{frame.height} does not match state {state.width}x{state.height}"
        )
    if t_now <= t_prev:
        raise ValueError(f"t_now ({t_now}) must be greater than t_prev ({t_prev})")


def _engine(state: PixelStateGrid, config: EventCameraConfig, order: int, dt: int) -> StepEngine:
    cap = int(config.capacity(state.width, state.height))
    if cap < 0:
        raise ValueError("max_events_per_frame must be >= 0")
    max_dt = 1 << max(1, int(dt - 1).bit_length())  # power-of-two bucket: fewer engines
    shape = StepShape(1, 1, state.height, state.width, cap, order, max_dt,
                      float(config.log_eps), int(config.refractory_us), state.uniform_thresholds)
    eng = state._ctx.get(shape)
    if eng is None:
        eng = StepEngine(shape, state.device)
        state._ctx[shape] = eng
    return eng


def run_generate(state: PixelStateGrid, frame: IntensityFrame, t_prev: int, t_now: int,
                 config: EventCameraConfig, order: int, stats=None, device_output: bool = False):
    """Shared body of generate_events_serial / generate_events_parallel."""
    _check_step(state, frame, t_prev, t_now)
    if config.log_eps <= 0:
        raise ValueError("log_eps must be positive")
    dt = int(t_now) - int(t_prev)
    if dt >= (1 << 31):
        raise ValueError("t_now - t_prev must be < 2**31 us")
    eng = _engine(state, config, order, dt)
    dframe = upload_frame(frame.values, state.device, state._ctx)
    eng.launch(dframe, state.d_ref_log, state.d_last_event_t, state.d_thresholds_pos,
               state.d_thresholds_neg, t_bounds=None, t0=int(t_prev), tick=dt, validate=True)
    counts, dropped, res, bad = eng.fetch_info()
    if bad != _lib.NO_BAD:
        eng.reset_bad()
        raise _bad_pixel_error(frame.values, bad, frame.width)
    n = int(counts[0])
    if stats is not None:
        stats.reservation_count = int(res[0]) if n + int(dropped[0]) > 0 else 0
        stats.events_emitted = n
    if device_output:
        out = DeviceEventBatch(eng.ev_t[0, :n].clone(), eng.ev_x[0, :n].clone(),
                               eng.ev_y[0, :n].clone(), eng.ev_p[0, :n].clone(),
                               dropped_count=int(dropped[0]), canonical=order == _lib.EVS_ORDER_CANONICAL)
        return out
    if n == 0:
        b = EventBatch.empty(dropped_count=int(dropped[0]))
    else:
        # fresh pinned host arrays (torch's caching host allocator recycles the
        # blocks once the caller drops the batch): one async copy each, one sync
        pool = state._ctx.setdefault("d2h_pool", PinnedPool())
        t, x, y, p = d2h_rows(pool, n, [eng.ev_t[0], eng.ev_x[0], eng.ev_y[0], eng.ev_p[0]])
        b = EventBatch(t=t.view(np.uint64), x=x.view(np.uint16), y=y.view(np.uint16), polarity=p,
                       dropped_count=int(dropped[0]), canonical=order == _lib.EVS_ORDER_CANONICAL)
    if stats is not None and getattr(stats, "collect_spans", False):
        stats.write_spans = _chunk_spans(b, state.width)
    return b


def _chunk_spans(b: EventBatch, width: int) -> list[tuple[int, int]]:
    """Write-once spans of the pixel-major placement: one (base, count) per
    active 32-pixel chunk, in chunk order (AggregationStats.write_spans)."""
    if len(b) == 0:
        return []
    pix = b.y.astype(np.int64) * width + b.x.astype(np.int64)
    chunk = pix // 32
    uniq, counts = np.unique(chunk, return_counts=True)
    bases = np.concatenate([[0], np.cumsum(counts)[:-1]])
    return [(int(a), int(c)) for a, c in zip(bases, counts)]


def generate_events_serial(state: PixelStateGrid, frame: IntensityFrame, t_prev: int, t_now: int,
                           config: EventCameraConfig) -> EventBatch:
    """model.py:79-171: pixel-major emission order (the definition's order).

    Mutates ``state`` in place (in HBM).
    """
    return run_generate(state, frame, t_prev, t_now, config, _lib.EVS_ORDER_PIXEL_MAJOR)


def inject_noise_events(width: int, height: int, t_prev: int, t_now: int, noise_rate_hz: float,
                        seed: int) -> EventBatch:
    """model.py:174-212: exact numpy-PCG64 background noise, generated on the GPU."""
    from ..noise import noise_events

    return noise_events(width, height, t_prev, t_now, noise_rate_hz, seed)


def limit_bandwidth(batch, max_events_per_sec: float, window_us: int):
    """model.py:215-246."""
    from ..represent import limit_bandwidth as _lb

    return _lb(batch, max_events_per_sec, window_us)


def accumulate_events_to_image(batch, window_us: int, t_end: int, width: int, height: int) -> np.ndarray:
    """model.py:249-262: signed polarity sum over t in [t_end - window, t_end)."""
    from ..represent import accumulate

    return accumulate(batch, window_us, t_end, width, height)
