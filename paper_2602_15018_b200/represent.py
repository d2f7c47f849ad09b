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


def merge_canonical(a: DeviceEventBatch, b: DeviceEventBatch) -> DeviceEventBatch:
    """Canonical order of concat([a, b]) for canonical a and b (merge, no sort)."""
    import torch

    L = _lib.load()
    na, nb = len(a), len(b)
    dev = a.t.device
    if nb == 0 or na == 0:
        src = a if nb == 0 else b
        return DeviceEventBatch(src.t, src.x, src.y, src.polarity, a.dropped_count + b.dropped_count, True)
    tmin = min(int(a.t[0].item()), int(b.t[0].item()))
    out = DeviceEventBatch(torch.empty(na + nb, dtype=torch.int64, device=dev),
                           torch.empty(na + nb, dtype=torch.int16, device=dev),
                           torch.empty(na + nb, dtype=torch.int16, device=dev),
                           torch.empty(na + nb, dtype=torch.int8, device=dev),
                           a.dropped_count + b.dropped_count, True)
    ws, _ep = _workspace(("merge", dev), nb * 8, dev)
    rc = L.evs_merge_canonical(na, a.t.data_ptr(), a.x.data_ptr(), a.y.data_ptr(), a.polarity.data_ptr(),
                               nb, b.t.data_ptr(), b.x.data_ptr(), b.y.data_ptr(), b.polarity.data_ptr(), tmin,
                               out.t.data_ptr(), out.x.data_ptr(), out.y.data_ptr(), out.polarity.data_ptr(),
                               ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    _lib.check(rc, "evs_merge_canonical")
    return out


def canonical_sort(batch):
    """parallel.py:112-123 on the GPU (stable order by t, y, x, polarity)."""
    _lib.require_cuda()
    if len(batch) == 0:
        return (EventBatch.empty(dropped_count=batch.dropped_count) if not isinstance(batch, DeviceEventBatch)
                else DeviceEventBatch(batch.t, batch.x, batch.y, batch.polarity, batch.dropped_count, True))
    if getattr(batch, "canonical", False):
        return batch
    parts = getattr(batch, "parts", None)
    if parts is not None and len(parts) == 2 and getattr(parts[0], "canonical", False):
        # concat_batches([signal (canonical), noise]): sort the small part, merge
        a, was_host = _device_batch(parts[0])
        b = canonical_sort(parts[1].to_device() if not isinstance(parts[1], DeviceEventBatch) else parts[1])
        sa = batch_stats(a) if len(a) else None
        sb = batch_stats(b) if len(b) else None
        if (sa and sb and sa[4] == 0 and sb[4] == 0 and min(sa[0], sb[0]) >= 0
                and max(sa[1], sb[1]) - min(sa[0], sb[0]) < (1 << 31)):
            out = merge_canonical(a, b)
            return out.to_host() if not isinstance(batch, DeviceEventBatch) else out
    db, was_host = _device_batch(batch)
    n = len(db)
    tmin, tmax, _xm, _ym, badp = batch_stats(db)
    span = tmax - tmin
    out = DeviceEventBatch(db.t.clone(), db.x.clone(), db.y.clone(), db.polarity.clone(),
                           dropped_count=db.dropped_count, canonical=True)
    L = _lib.load()
    if badp or span >= (1 << 31) or tmin < 0:
        # outside the simulator's range (polarity not +-1, uint64 times >= 2^63
        # or spanning >= 2^31 us): the general four-pass sort
        if n >= (1 << 32):
            raise ValueError("canonical_sort on the GPU handles < 2**32 events per batch")
        ws, _ep = _workspace(("sort_general", db.t.device), L.evs_sort_general_workspace_bytes(n), db.t.device)
        rc = L.evs_canonical_sort_general(n, out.t.data_ptr(), out.x.data_ptr(), out.y.data_ptr(),
                                          out.polarity.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
        _lib.check(rc, "evs_canonical_sort_general")
        return out.to_host() if was_host else out
    nbytes = L.evs_sort_workspace_bytes(n, span)
    ws, ep = _workspace(("sort", db.t.device), nbytes, db.t.device)
    rc = L.evs_canonical_sort(n, out.t.data_ptr(), out.x.data_ptr(), out.y.data_ptr(),
                              out.polarity.data_ptr(), tmin, span, ep.take(ws),
                              ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel()),
                              ctypes.c_void_p(_lib.stream_ptr()))
    _lib.check(rc, "evs_canonical_sort")
    return out.to_host() if was_host else out


def accumulate(batch, window_us: int, t_end: int, width: int, height: int, device_output: bool = False):
    """accumulate_events_to_image (model.py:249-262) on the GPU; int64 (H, W)."""
    import torch

    _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    if len(batch):
        db, _ = _device_batch(batch)
        _tmin, _tmax, xm, ym, _badp = batch_stats(db)
        if xm >= width or ym >= height:  # model.py:253-254
            raise ValueError("event coordinates out of bounds for the given dimensions")
    grid = torch.empty((height, width), dtype=torch.int64, device=dev)
    L = _lib.load()
    if len(batch) == 0:
        grid.zero_()
    else:
        rc = L.evs_accumulate(len(db), db.t.data_ptr(), db.x.data_ptr(), db.y.data_ptr(), db.polarity.data_ptr(),
                              int(window_us), int(t_end), int(width), int(height), grid.data_ptr(),
                              _lib.stream_ptr())
        _lib.check(rc, "evs_accumulate")
    return grid if device_output else grid.cpu().numpy()


def voxel_grid(batch, t0: int, t1: int, width: int, height: int, bins: int = 5, device_output: bool = False):
    """Voxel grid of the events with t in [t0, t1) (repo-defined): f32 (bins, H, W)."""
    import torch

    _lib.require_cuda()
    if t1 <= t0 or bins < 2:
        raise ValueError("need t1 > t0 and bins >= 2")
    dev = torch.device("cuda", torch.cuda.current_device())
    L = _lib.load()
    out = torch.empty((bins, height, width), dtype=torch.float32, device=dev)
    if len(batch):
        db, _ = _device_batch(batch)
        _tmin, _tmax, xm, ym, _badp = batch_stats(db)
        if xm >= width or ym >= height:
            raise ValueError("event coordinates out of bounds for the given dimensions")
        n, tp, xp, yp, pp = len(db), db.t.data_ptr(), db.x.data_ptr(), db.y.data_ptr(), db.polarity.data_ptr()
    else:
        n, tp, xp, yp, pp = 0, None, None, None, None
    nbytes = L.evs_voxel_workspace_bytes(bins, width, height)
    ws, _ep = _workspace(("voxel", dev), nbytes, dev)
    rc = L.evs_voxel(n, tp, xp, yp, pp, int(t0), int(t1), int(bins), int(width), int(height), out.data_ptr(),
                     ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    _lib.check(rc, "evs_voxel")
    return out if device_output else out.cpu().numpy()


def limit_bandwidth(batch, max_events_per_sec: float, window_us: int):
    """limit_bandwidth (model.py:215-246) on the GPU."""
    import torch

    if window_us <= 0:
        raise ValueError("window_us must be positive")
    if max_events_per_sec < 0:
        raise ValueError("max_events_per_sec must be >= 0")
    if len(batch) == 0:
        if isinstance(batch, DeviceEventBatch):
            return DeviceEventBatch(batch.t[:0], batch.x[:0], batch.y[:0], batch.polarity[:0],
                                    batch.dropped_count, True)
        return EventBatch.empty(dropped_count=batch.dropped_count)
    _lib.require_cuda()
    db, was_host = _device_batch(batch)
    n = len(db)
    cap = int(max_events_per_sec * window_us * 1e-6)  # model.py:233
    L = _lib.load()
    dev = db.t.device
    ot = torch.empty(n, dtype=torch.int64, device=dev)
    ox = torch.empty(n, dtype=torch.int16, device=dev)
    oy = torch.empty(n, dtype=torch.int16, device=dev)
    op = torch.empty(n, dtype=torch.int8, device=dev)
    meta = torch.empty(2, dtype=torch.int64, device=dev)
    ws, _ep = _workspace(("lb", dev), L.evs_limit_bandwidth_workspace_bytes(n), dev)
    rc = L.evs_limit_bandwidth(n, db.t.data_ptr(), db.x.data_ptr(), db.y.data_ptr(), db.polarity.data_ptr(),
                               cap, int(window_us), ot.data_ptr(), ox.data_ptr(), oy.data_ptr(), op.data_ptr(),
                               meta.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    _lib.check(rc, "evs_limit_bandwidth")
    kept, unsorted = meta.cpu().tolist()
    if unsorted:
        raise ValueError("limit_bandwidth requires a timestamp-sorted batch")
    out = DeviceEventBatch(ot[:kept], ox[:kept], oy[:kept], op[:kept],
                           dropped_count=int(batch.dropped_count) + (n - kept),
                           canonical=getattr(batch, "canonical", False))
    return out.to_host() if was_host else out
