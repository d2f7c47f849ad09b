"""Device-side batch operations: canonical sort, histogram / voxel binning,
bandwidth limiting.  Thin host wrappers over the C ABI; no CPU fallback."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .events.types import DeviceEventBatch, EventBatch

_sort_ctx: dict = {}


def _device_batch(batch) -> tuple[DeviceEventBatch, bool]:
    if isinstance(batch, DeviceEventBatch):
        return batch, False
    return batch.to_device(), True


def _workspace(key, nbytes: int, device):
    import torch

    ws = _sort_ctx.get(key)
    if ws is None or ws.numel() < nbytes or ws.device != device:
        ws = torch.zeros(max(int(nbytes), 1), dtype=torch.uint8, device=device)
        _sort_ctx[key] = ws
        _sort_ctx[(key, "epoch")] = _lib.EpochCounter()
    return ws, _sort_ctx[(key, "epoch")]


def batch_stats(db: DeviceEventBatch):
    """(t_min, t_max, x_max, y_max, bad_polarity) of a device batch (synchronising)."""
    import torch

    L = _lib.load()
    out = torch.empty(5, dtype=torch.int64, device=db.t.device)
    rc = L.evs_batch_stats(len(db), db.t.data_ptr(), db.x.data_ptr(), db.y.data_ptr(),
                           db.polarity.data_ptr(), out.data_ptr(), _lib.stream_ptr())
    _lib.check(rc, "evs_batch_stats")
    return [int(v) for v in out.cpu().tolist()]


def canonical_sort(batch):
    """parallel.py:112-123 on the GPU (stable order by t, y, x, polarity)."""
    _lib.require_cuda()
    if len(batch) == 0:
        return (EventBatch.empty(dropped_count=batch.dropped_count) if not isinstance(batch, DeviceEventBatch)
                else DeviceEventBatch(batch.t, batch.x, batch.y, batch.polarity, batch.dropped_count, True))
    if getattr(batch, "canonical", False):
        return batch
    db, was_host = _device_batch(batch)
    n = len(db)
    tmin, tmax, _xm, _ym, badp = batch_stats(db)
    span = tmax - tmin
    if badp or span >= (1 << 31) or tmin < 0:
        raise NotImplementedError("canonical_sort on the GPU needs polarity in {-1,+1}, "
                                  "0 <= t and max(t)-min(t) < 2**31")
    out = DeviceEventBatch(db.t.clone(), db.x.clone(), db.y.clone(), db.polarity.clone(),
                           dropped_count=db.dropped_count, canonical=True)
    L = _lib.load()
    nbytes = L.evs_sort_workspace_bytes(n, span)
    ws, ep = _workspace(("sort", db.t.device), nbytes, db.t.device)
    rc = L.evs_canonical_sort(n, out.t.data_ptr(), out.x.data_ptr(), out.y.data_ptr(),
                              out.polarity.data_ptr(), tmin, span, ep.take(ws),
                              ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel()),
                              ctypes.c_void_p(_lib.stream_ptr()))
    _lib.check(rc, "evs_canonical_sort")
    return out.to_host() if was_host else out


def accumulate(batch, window_us: int, t_end: int, width: int, height: int) -> np.ndarray:
    raise NotImplementedError("accumulate: GPU kernel not built yet")


def limit_bandwidth(batch, max_events_per_sec: float, window_us: int):
    raise NotImplementedError("limit_bandwidth: GPU kernel not built yet")
