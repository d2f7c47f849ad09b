"""Row-band split of one large sensor across ranks.

north_star: "work is partitioned ... by independent camera/environment
streams, with a spatial row-band split for single very large sensors".
Pixels are independent, so rank r simulates rows [y0_r, y1_r) of the camera
with its own slice of the pixel state (``GpuBand``: the ``evs_step`` kernels
on that slice, canonical order, y shifted to sensor rows).  The only
exchanges are per frame an all_gather of five int64 per band (events
generated, events kept, reservations, first invalid pixel, its value) and,
where a consumer needs the frame on one rank, ``gather_keys`` of the packed
8-byte keys (``distributed.py``; written by the evs_pack_segments kernel) and
one k-way merge of the bands' sorted runs on that rank (evs_merge_runs).

The result equals the unsplit reference (model.py:79-171, parallel.py:126-273
followed by canonical_sort, parallel.py:112-123):

* order: each band's keys (t_rel << 33 | y << 17 | x << 1 | p) are sorted and
  key order is the canonical (t, y, x, p) order, so the sensor's batch is the
  sorted union of the bands' keys;
* reservation_count: band starts are multiples of 32 pixels in row-major
  order (``band_rows``), so no 32-pixel chunk (parallel.py:219-225) straddles
  two bands and the per-band counts add up;
* capacity: the reference keeps the first ``cap`` events in pixel-major order
  (model.py:150-158).  Band b may keep ``cap - (events of bands < b)``; a band
  whose share is smaller than what it kept re-runs the frame from its
  pre-frame state in pixel-major order and keeps that prefix (only frames
  above the capacity pay for this; the state update does not depend on the
  capacity);
* invalid frames: the reference raises before mutating (model.py:33-38); a
  band that saw a bad pixel leaves its state untouched, every band restores
  its pre-frame state, and every rank raises the ValueError of the first bad
  pixel in row-major order over the whole sensor.

``BandedCamera`` drives one band per rank through a communicator
(``TorchComm`` = torch.distributed, NCCL on GPUs, gloo in the CPU tests);
``LocalBands`` runs several bands in one process with the same planning
functions (parity tests on one GPU).
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .events.types import DeviceEventBatch, EventBatch, EventCameraConfig, PixelStateGrid

NO_BAD = _lib.NO_BAD


def band_rows(height: int, width: int, nbands: int) -> list[tuple[int, int]]:
    """Row ranges [y0, y1) of ``nbands`` bands, as equal as possible, every
    band start a multiple of 32 pixels in row-major order (y0 * width % 32 == 0).
    Bands may be empty when the sensor has fewer row groups than bands."""
    if nbands < 1 or height < 0 or width < 1:
        raise ValueError("band_rows: need nbands >= 1, height >= 0, width >= 1")
    g = 32 // math.gcd(width, 32)  # row granularity
    groups = -(-height // g)
    out = []
    for b in range(nbands):
        y0 = min(height, (b * groups // nbands) * g)
        y1 = min(height, ((b + 1) * groups // nbands) * g)
        out.append((y0, y1))
    return out


@dataclass
class BandResult:
    """One band's frame: ``keys`` sorted int64 (sensor rows, t relative to t_prev)."""
    total: int          # events generated (kept by refractory) in the band
    written: int        # events the band holds in ``keys``
    reservations: int   # 32-pixel chunks with >= 1 event
    bad: int            # first invalid pixel as a SENSOR flat index, or NO_BAD
    bad_bits: int       # float32 bits of that pixel's value (0 if none)
    keys: object        # torch int64 [written]


@dataclass
class FramePlan:
    bad: int
    bad_bits: int
    allowed: list       # events each band may keep
    rerun: list         # bands that must redo the frame with a smaller share
    written: int
    dropped: int
    reservations: int


def plan_frame(stats: list, cap: int) -> FramePlan:
    """Combine per-band (total, written, reservations, bad, bad_bits) rows,
    bands in row order, into the sensor's frame outcome."""
    bads = [(int(s[3]), int(s[4])) for s in stats if int(s[3]) != NO_BAD]
    bad, bad_bits = min(bads) if bads else (NO_BAD, 0)
    totals = [int(s[0]) for s in stats]
    allowed, rerun = [], []
    pre = 0
    for b, s in enumerate(stats):
        share = max(0, min(totals[b], cap - pre))
        allowed.append(share)
        if share < int(s[1]):
            rerun.append(b)
        pre += totals[b]
    total = sum(totals)
    written = min(total, cap)
    res = sum(int(s[2]) for s in stats)
    return FramePlan(bad, bad_bits, allowed, rerun, written, total - written, res if total > 0 else 0)


def bad_pixel_error(flat: int, bits: int, width: int) -> ValueError:
    yy, xx = divmod(int(flat), width)
    val = np.float32(struct.unpack("<f", struct.pack("<I", int(bits) & 0xFFFFFFFF))[0])
    return ValueError(f"invalid intensity {val!r} at pixel (x={xx}, y={yy})")


def merge_keys(keys, counts):
    """Sensor order from the bands' sorted key runs (band order, ``counts``
    keys each): the evs_merge_runs kernel (key order is canonical, and a
    band's rows all precede the next band's, so this is SURVEY.md 8(e)'s
    (t, band) placement)."""
    import torch

    if keys.numel() == 0 or len(counts) == 1:
        return keys
    offs = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int64, device=keys.device)
    out = torch.empty_like(keys)
    rc = _lib.load().evs_merge_runs(len(counts), offs.data_ptr(), keys.numel(), keys.data_ptr(), out.data_ptr(),
                                    _lib.stream_ptr())
    _lib.check(rc, "evs_merge_runs")
    return out


def keys_to_batch(keys, t_prev: int, dropped: int, device_output: bool = False):
    from .distributed import KEY64_LAYOUT, unpack_keys

    t, x, y, p = unpack_keys(keys, int(t_prev), KEY64_LAYOUT)
    if device_output:
        return DeviceEventBatch(t, x.short(), y.short(), p, dropped_count=int(dropped),
                                canonical=True)
    if keys.numel() == 0:
        return EventBatch.empty(dropped_count=int(dropped))
    return EventBatch(t=t.cpu().numpy().view(np.uint64), x=x.cpu().numpy().astype(np.uint16),
                      y=y.cpu().numpy().astype(np.uint16), polarity=p.cpu().numpy(),
                      dropped_count=int(dropped), canonical=True)


class GpuBand:
    """Rows [y0, y1) of one sensor on this rank's GPU (the evs_step kernels)."""

    def __init__(self, state: PixelStateGrid, rows: tuple, config: EventCameraConfig, device=None):
        """``state``: the WHOLE sensor's initial state (init_pixel_states: the
        threshold draws are the sensor's); only the band's rows are kept."""
        import torch

        self.y0, self.y1 = int(rows[0]), int(rows[1])
        self.width, self.height = state.width, self.y1 - self.y0
        self.sensor_height = state.height
        self.config = config
        self.cap = int(config.capacity(state.width, state.height))
        dev = device or torch.device("cuda", torch.cuda.current_device())
        sl = slice(self.y0, self.y1)
        uni = state.uniform_thresholds
        # the band owns a copy of its rows (not a view of the sensor's grid)
        self.state = PixelStateGrid(
            self.width, self.height, state.d_ref_log[sl].to(dev).clone(),
            state.d_last_event_t[sl].to(dev).clone(),
            (np.full((self.height, self.width), uni[0], np.float32) if uni
             else state.d_thresholds_pos[sl].to(dev).clone()),
            (np.full((self.height, self.width), uni[1], np.float32) if uni
             else state.d_thresholds_neg[sl].to(dev).clone()),
            device=dev)
        self.device = dev
        self._saved = None
        self._engines = {}

    def _engine(self, order: int, dt: int):
        from .runtime import StepEngine, StepShape

        max_dt = 1 << max(1, int(dt - 1).bit_length())
        shape = StepShape(1, 1, self.height, self.width, self.cap, order, max_dt,
                          float(self.config.log_eps), int(self.config.refractory_us),
                          self.state.uniform_thresholds)
        eng = self._engines.get(shape)
        if eng is None:
            eng = self._engines[shape] = StepEngine(shape, self.device)
        return eng

    def band_frame(self, frame):
        """The band's rows of a full-sensor frame (host or device), or a band-shaped frame."""
        import torch

        v = frame.values if hasattr(frame, "values") else frame
        t = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v, np.float32))
        if t.shape[0] == self.sensor_height and self.height != self.sensor_height:
            t = t[self.y0:self.y1]
        if tuple(t.shape) != (self.height, self.width):
            raise ValueError(f"frame rows {tuple(t.shape)} do not match band {self.height}x{self.width}")
        return t.to(device=self.device, dtype=torch.float32).contiguous()

    def save(self) -> None:
        s = self.state
        if self._saved is None:
            self._saved = (s.d_ref_log.clone(), s.d_last_event_t.clone())
        else:
            self._saved[0].copy_(s.d_ref_log)
            self._saved[1].copy_(s.d_last_event_t)

    def restore(self) -> None:
        self.state.d_ref_log.copy_(self._saved[0])
        self.state.d_last_event_t.copy_(self._saved[1])

    def run(self, frame_band, t_prev: int, t_now: int, keep: int | None = None) -> BandResult:
        """One frame of the band.  keep=None: canonical order, the band's own
        capacity; keep=k: pixel-major order, the first k events (then sorted)."""
        import torch

        from .distributed import KEY64_LAYOUT, pack_segments
        from .represent import canonical_sort

        if self.height == 0:
            return BandResult(0, 0, 0, NO_BAD, 0, torch.empty(0, dtype=torch.int64, device=self.device))
        dt = int(t_now) - int(t_prev)
        order = _lib.EVS_ORDER_CANONICAL if keep is None else _lib.EVS_ORDER_PIXEL_MAJOR
        eng = self._engine(order, dt)
        s = self.state
        eng.launch(frame_band, s.d_ref_log, s.d_last_event_t, s.d_thresholds_pos, s.d_thresholds_neg,
                   t0=int(t_prev), tick=dt, validate=True)
        counts, dropped, res, bad = eng.fetch_info()
        if bad != NO_BAD:
            eng.reset_bad()
            v = float(frame_band.reshape(-1)[bad].item())
            bits = struct.unpack("<I", struct.pack("<f", v))[0]
            return BandResult(0, 0, 0, bad + self.y0 * self.width, bits,
                              torch.empty(0, dtype=torch.int64, device=self.device))
        n = int(counts[0])
        total = n + int(dropped[0])
        if keep is not None:
            n = min(n, int(keep))
        rows = (eng.ev_t, eng.ev_x, eng.ev_y, eng.ev_p)
        cnt = eng.info[0, :1]
        if keep is not None and n > 0:  # the first `keep` pixel-major events, then canonical order
            b = canonical_sort(DeviceEventBatch(eng.ev_t[0, :n], eng.ev_x[0, :n], eng.ev_y[0, :n], eng.ev_p[0, :n]))
            rows = (b.t[None], b.x[None], b.y[None], b.polarity[None])
            cnt = torch.tensor([n], dtype=torch.int64, device=self.device)
        # 8-byte keys (t - t_prev) << 33 | sensor row << 17 | x << 1 | p, written by the evs_pack_segments kernel
        keys, _ = pack_segments(cnt, rows, int(t_prev), KEY64_LAYOUT, 8, y_offset=self.y0)
        return BandResult(total, n, int(res[0]), NO_BAD, 0, keys[:n])


class TorchComm:
    """The two exchanges over torch.distributed (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device

    def all_gather_stats(self, row: list, device) -> list:
        import torch
        import torch.distributed as dist

        t = torch.tensor(row, dtype=torch.int64, device=device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return [[int(v) for v in o.tolist()] for o in out]

    def gather_keys(self, keys, dst: int):
        """(keys of every band back to back in band order, per-band counts) on dst."""
        from .distributed import gather_keys

        return gather_keys(keys.contiguous(), dst=dst, group=self.group)


class BandedCamera:
    """One sensor split into row bands, band ``comm.rank`` on this rank.

    ``step`` returns the sensor's canonical EventBatch on ``dst`` (None on the
    other ranks, or on every rank with gather=False) and fills ``stats``
    (reservation_count, events_emitted) like generate_events_parallel."""

    def __init__(self, band, comm, config: EventCameraConfig, sensor_width: int, sensor_height: int,
                 merge=merge_keys):
        self.band, self.comm, self.config = band, comm, config
        self.width, self.height = int(sensor_width), int(sensor_height)
        self.cap = int(config.capacity(self.width, self.height))
        self.merge = merge  # (keys, per-band counts) -> merged keys (the kernel; CPU tests pass a stand-in)

    def step(self, frame, t_prev: int, t_now: int, stats=None, dst: int = 0, gather: bool = True,
             device_output: bool = False):
        if int(t_now) <= int(t_prev):
            raise ValueError(f"t_now ({t_now}) must be greater than t_prev ({t_prev})")
        band = self.band
        fb = band.band_frame(frame)
        band.save()
        r = band.run(fb, t_prev, t_now)
        rows = self.comm.all_gather_stats([r.total, r.written, r.reservations, r.bad, r.bad_bits],
                                          r.keys.device)
        plan = plan_frame(rows, self.cap)
        if plan.bad != NO_BAD:
            band.restore()
            raise bad_pixel_error(plan.bad, plan.bad_bits, self.width)
        me = self.comm.rank
        if me in plan.rerun:
            band.restore()
            r = band.run(fb, t_prev, t_now, keep=plan.allowed[me])
        if stats is not None:
            stats.reservation_count = plan.reservations
            stats.events_emitted = plan.written
        if not gather:
            return None
        keys, counts = self.comm.gather_keys(r.keys, dst)
        if me != dst:
            return None
        return keys_to_batch(self.merge(keys, counts), t_prev, plan.dropped, device_output)


class LocalBands:
    """Several bands of one sensor in one process (same planning as BandedCamera)."""

    def __init__(self, bands: list, config: EventCameraConfig, sensor_width: int, sensor_height: int):
        self.bands, self.config = bands, config
        self.width, self.height = int(sensor_width), int(sensor_height)
        self.cap = int(config.capacity(self.width, self.height))

    def step(self, frame, t_prev: int, t_now: int, stats=None, device_output: bool = False):
        import torch

        if int(t_now) <= int(t_prev):
            raise ValueError(f"t_now ({t_now}) must be greater than t_prev ({t_prev})")
        fbs = [b.band_frame(frame) for b in self.bands]
        for b in self.bands:
            b.save()
        res = [b.run(fb, t_prev, t_now) for b, fb in zip(self.bands, fbs)]
        plan = plan_frame([[r.total, r.written, r.reservations, r.bad, r.bad_bits] for r in res], self.cap)
        if plan.bad != NO_BAD:
            for b in self.bands:
                b.restore()
            raise bad_pixel_error(plan.bad, plan.bad_bits, self.width)
        for i in plan.rerun:
            self.bands[i].restore()
            res[i] = self.bands[i].run(fbs[i], t_prev, t_now, keep=plan.allowed[i])
        if stats is not None:
            stats.reservation_count = plan.reservations
            stats.events_emitted = plan.written
        keys = torch.cat([r.keys.to(res[0].keys.device) for r in res])
        return keys_to_batch(merge_keys(keys, [int(r.keys.numel()) for r in res]), t_prev, plan.dropped,
                             device_output)
