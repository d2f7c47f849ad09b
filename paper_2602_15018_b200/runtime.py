"""Host runtime around the C ABI: workspaces, output pools, epochs, streams.

``StepEngine`` owns everything one ``evs_step`` shape needs (device
workspace, padded per-segment output pool, per-segment counters) so repeated
calls allocate nothing.  All work is enqueued on the caller's CUDA stream;
nothing here synchronises except the explicit ``fetch_*`` helpers.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class StepShape:
    streams: int
    frames: int
    height: int
    width: int
    capacity: int
    order: int
    max_dt: int
    log_eps: float
    refractory_us: int
    uniform: tuple | None  # (th_pos, th_neg) or None


class StepEngine:
    """Reusable launch context for one StepShape (one sensor group)."""

    def __init__(self, shape: StepShape, device):
        import torch

        if int(shape.refractory_us) >= (1 << 30):
            # the kernels compare refractory periods in int32 against last-event
            # times clamped to +-2^30 us around the frame start
            raise ValueError("refractory_us must be < 2**30 us (about 17.9 minutes) on the GPU path")
        _lib.require_cuda()
        self.shape = shape
        self.device = device
        self.lib = _lib.load()
        self.params = _lib.StepParams()
        p = self.params
        p.streams, p.frames = shape.streams, shape.frames
        p.height, p.width = shape.height, shape.width
        p.log_eps = float(shape.log_eps)
        p.refractory_us = int(shape.refractory_us)
        p.capacity = int(shape.capacity)
        if shape.uniform is not None:
            p.th_pos_uniform, p.th_neg_uniform = shape.uniform
        p.max_dt = int(shape.max_dt)
        p.order = int(shape.order)
        p.validate = 1
        nbytes = self.lib.evs_step_workspace_bytes(ctypes.byref(p))
        if nbytes == 0:
            raise ValueError(f"unsupported step shape {shape}")
        self.workspace = torch.zeros(int(nbytes), dtype=torch.uint8, device=device)
        nseg = shape.streams * shape.frames
        cap = max(int(shape.capacity), 1)
        self.ev_t = torch.empty((nseg, cap), dtype=torch.int64, device=device)
        self.ev_x = torch.empty((nseg, cap), dtype=torch.int16, device=device)
        self.ev_y = torch.empty((nseg, cap), dtype=torch.int16, device=device)
        self.ev_p = torch.empty((nseg, cap), dtype=torch.int8, device=device)
        # info rows: counts, dropped, reservations ; bad pixel in a separate slot
        self.info = torch.zeros((3, nseg), dtype=torch.int64, device=device)
        self.bad = torch.full((1,), _lib.NO_BAD, dtype=torch.int64, device=device)
        self.epochs = _lib.EpochCounter()
        self.bufs = _lib.StepBuffers()

    def launch(self, frames, ref_log, last_event_t, th_pos=None, th_neg=None, t_bounds=None,
               t0: int = 0, tick: int = 0, validate: bool = True, stream=None,
               stage_events=None) -> None:
        """Enqueue one evs_step on `stream` (default: torch's current stream).

        stage_events: optional list of 5 torch.cuda.Event(enable_timing=True)
        recorded around the prologue / generate / plan / order stages.
        """
        p, b = self.params, self.bufs
        p.t0, p.tick = int(t0), int(tick)
        p.validate = 1 if validate else 0
        p.epoch = self.epochs.take(self.workspace)
        b.frames = frames.data_ptr()
        b.t_bounds = t_bounds.data_ptr() if t_bounds is not None else None
        b.ref_log = ref_log.data_ptr()
        b.last_event_t = last_event_t.data_ptr()
        if self.shape.uniform is None:
            b.th_pos, b.th_neg = th_pos.data_ptr(), th_neg.data_ptr()
        else:
            b.th_pos = b.th_neg = None
        b.ev_t, b.ev_x = self.ev_t.data_ptr(), self.ev_x.data_ptr()
        b.ev_y, b.ev_p = self.ev_y.data_ptr(), self.ev_p.data_ptr()
        b.counts = self.info[0].data_ptr()
        b.dropped = self.info[1].data_ptr()
        b.reservations = self.info[2].data_ptr()
        b.bad_pixel = self.bad.data_ptr()
        ws = ctypes.c_void_p(self.workspace.data_ptr())
        nb = ctypes.c_size_t(self.workspace.numel())
        sp = ctypes.c_void_p(_lib.stream_ptr(stream))
        if stage_events is None:
            rc = self.lib.evs_step(ctypes.byref(p), ctypes.byref(b), ws, nb, sp)
        else:
            handles = (ctypes.c_void_p * len(stage_events))(*[e.cuda_event for e in stage_events])
            rc = self.lib.evs_step_profiled(ctypes.byref(p), ctypes.byref(b), ws, nb, sp, handles,
                                            len(stage_events))
        _lib.check(rc, "evs_step")

    # -- CUDA-graph replay with the device-resident step clock ----------------
    def capture(self, windows, ref_log, last_event_t, th_pos=None, th_neg=None, tick: int = 1000,
                t0: int = 0, validate: bool = True):
        """Capture one CUDA graph running one step per frame window (in order).

        Start times and lookback epochs advance on the device
        (EVS_FLAG_DEVICE_CLOCK), so ``replay()`` continues the sequence: replay
        r covers frames [r*len(windows)*T, (r+1)*len(windows)*T) after t0.
        """
        import torch

        p = self.params
        p.flags = _lib.EVS_FLAG_DEVICE_CLOCK
        p.tick = int(tick)
        self._graph_steps = len(windows)
        self._clock_tick = int(tick)
        self._clock_t0 = int(t0)
        # (callers run eager steps first so kernel attributes are already set)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(self.graph, stream=s):
                for win in windows:
                    self._launch_dc(win, ref_log, last_event_t, th_pos, th_neg, validate)
        torch.cuda.current_stream().wait_stream(s)
        p.flags = 0
        self._graph_args = (ref_log, last_event_t, th_pos, th_neg, windows)

    def _clock_set(self, t0: int, epoch: int):
        """Point the device clock at (t0, epoch); flags must include DEVICE_CLOCK for sizing."""
        rc = self.lib.evs_step_clock_init(ctypes.byref(self.params), ctypes.c_void_p(self.workspace.data_ptr()),
                                          ctypes.c_size_t(self.workspace.numel()), int(t0), int(epoch),
                                          ctypes.c_void_p(_lib.stream_ptr()))
        _lib.check(rc, "evs_step_clock_init")

    def _launch_dc(self, frames, ref_log, last_event_t, th_pos, th_neg, validate, stream=None, events=None):
        p, b = self.params, self.bufs
        p.validate = 1 if validate else 0
        b.frames = frames.data_ptr()
        b.t_bounds = None
        b.ref_log, b.last_event_t = ref_log.data_ptr(), last_event_t.data_ptr()
        if self.shape.uniform is None:
            b.th_pos, b.th_neg = th_pos.data_ptr(), th_neg.data_ptr()
        else:
            b.th_pos = b.th_neg = None
        b.ev_t, b.ev_x = self.ev_t.data_ptr(), self.ev_x.data_ptr()
        b.ev_y, b.ev_p = self.ev_y.data_ptr(), self.ev_p.data_ptr()
        b.counts, b.dropped = self.info[0].data_ptr(), self.info[1].data_ptr()
        b.reservations, b.bad_pixel = self.info[2].data_ptr(), self.bad.data_ptr()
        ws, nb = ctypes.c_void_p(self.workspace.data_ptr()), ctypes.c_size_t(self.workspace.numel())
        sp = ctypes.c_void_p(_lib.stream_ptr(stream))
        if events is None:
            rc = self.lib.evs_step(ctypes.byref(p), ctypes.byref(b), ws, nb, sp)
        else:
            handles = (ctypes.c_void_p * len(events))(*[e.cuda_event if e is not None else None for e in events])
            rc = self.lib.evs_step_profiled(ctypes.byref(p), ctypes.byref(b), ws, nb, sp, handles, len(events))
        _lib.check(rc, "evs_step")

    def replay(self) -> None:
        """Replay the captured graph on the current stream (no host sync)."""
        # The graph's steps share the engine's epoch sequence with eager
        # launches, so stale lookback words can never carry a live epoch.
        need = self._graph_steps * _lib.EVS_EPOCHS_PER_CALL
        if self.epochs.value + need > _lib.EVS_EPOCH_LIMIT:
            self.workspace.zero_()
            self.epochs.value = 1
        self._clock_set(self._clock_t0, self.epochs.value)
        self.graph.replay()
        self.epochs.value += need
        self._clock_t0 += self._graph_steps * self.shape.frames * self._clock_tick

    def fetch_info(self):
        """Synchronising read of (counts, dropped, reservations, bad)."""
        import torch

        host = torch.cat([self.info.reshape(-1), self.bad]).cpu().numpy()
        nseg = self.info.shape[1]
        # the next calls' tile groups follow this call's event density (keys_hint:
        # performance only, the results do not depend on it)
        if int(host[-1]) == _lib.NO_BAD and nseg:
            self.params.keys_hint = int(max(0, int(host[:nseg].sum())) // nseg)
        if int(host[-1]) == _lib.NO_BAD and (host[nseg:2 * nseg] == -2).any():
            raise _lib.NativeError("a pixel would cross more than 2**20 thresholds in one frame: an infinite "
                                   "intensity (with validate=False) or a reference level (ref_log) far outside "
                                   "the log range of [0, 1] intensities")
        return host[:nseg], host[nseg:2 * nseg], host[2 * nseg:3 * nseg], int(host[-1])

    def reset_bad(self) -> None:
        self.bad.fill_(_lib.NO_BAD)


class PipelinedSteps:
    """Frame-by-frame stepping with consecutive steps overlapped: two
    StepEngines of one shape (two workspaces and two output pools) alternate on
    two streams, and step i+1 waits only for step i's K1 (the kernel that
    writes the pixel state) -- its K1 then runs while step i's histogram,
    scan and ordering kernels finish.  Used for one-frame steps (the
    reference's per-frame call granularity), where every kernel is a single
    partial wave.  Captured as one CUDA graph of an even number of steps with
    each engine's clock advancing two steps per call (clock_stride = 2);
    after a replay, step i's outputs are in engines[i % 2] until step i + 2.
    """

    def __init__(self, shape: StepShape, device):
        self.engines = [StepEngine(shape, device), StepEngine(shape, device)]
        self.shape = shape

    def capture(self, windows, ref_log, last_event_t, th_pos=None, th_neg=None, tick: int = 1000, t0: int = 0,
                validate: bool = True):
        import torch

        if len(windows) % 2:
            raise ValueError("PipelinedSteps captures an even number of steps")
        for e in self.engines:
            e.params.flags = _lib.EVS_FLAG_DEVICE_CLOCK
            e.params.tick = int(tick)
            e.params.clock_stride = 2
            e.params.keys_hint = max(x.params.keys_hint for x in self.engines)
        self._tick, self._t0, self._n = int(tick), int(t0), len(windows)
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        k1_done = [torch.cuda.Event() for _ in windows]
        for ev in k1_done:  # materialise the handles outside the capture
            ev.record()
        origin = torch.cuda.Stream()
        origin.wait_stream(torch.cuda.current_stream())
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=origin):
            for st in streams:
                st.wait_stream(origin)
            for i, win in enumerate(windows):
                st = streams[i % 2]
                if i > 0:
                    st.wait_event(k1_done[i - 1])
                self.engines[i % 2]._launch_dc(win, ref_log, last_event_t, th_pos, th_neg, validate, stream=st,
                                               events=[None, None, k1_done[i], None, None])
            for st in streams:
                origin.wait_stream(st)
        torch.cuda.current_stream().wait_stream(origin)
        for e in self.engines:
            e.params.flags = 0
            e.params.clock_stride = 0
        self._args = (windows, k1_done, streams)

    def replay(self) -> None:
        need = (self._n // 2) * _lib.EVS_EPOCHS_PER_CALL
        for j, e in enumerate(self.engines):
            if e.epochs.value + need > _lib.EVS_EPOCH_LIMIT:
                e.workspace.zero_()
                e.epochs.value = 1
            e.params.flags = _lib.EVS_FLAG_DEVICE_CLOCK
            e._clock_set(self._t0 + j * self.shape.frames * self._tick, e.epochs.value)
            e.params.flags = 0
        self.graph.replay()
        for e in self.engines:
            e.epochs.value += need
        self._t0 += self._n * self.shape.frames * self._tick


class PinnedPool:
    """Reusable pinned host blocks for device->host result copies.

    Results are handed out as numpy views into a block; a block is reused
    only once no view of it is alive (the views keep the block's root array
    referenced), so returned arrays stay valid for as long as the caller holds
    them -- the same ownership the reference's freshly allocated arrays have.
    """

    def __init__(self, keep: int = 8):
        self.roots = []  # (pinned uint8 tensor, its numpy root array)
        self.keep = keep

    def take(self, nbytes: int):
        import sys

        import torch

        for i, (t, r) in enumerate(self.roots):
            if r.nbytes >= nbytes and sys.getrefcount(r) <= 3:  # list tuple + r + the call
                return t, r
        size = 1 << 20
        while size < nbytes:  # power-of-two blocks: varying batch sizes reuse them
            size <<= 1
        t = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        r = t.numpy()
        self.roots.append((t, r))
        if len(self.roots) > self.keep:  # forget the oldest idle block
            for i, (_t, rr) in enumerate(self.roots[:-1]):
                if sys.getrefcount(rr) <= 3:
                    del self.roots[i]
                    break
        return t, r


def d2h_rows(pool: PinnedPool, n: int, rows, stream=None):
    """Copy the first n elements of each device tensor in `rows` into one pinned
    block (async copies, one synchronize); returns numpy views into it."""
    import torch

    sizes = [n * r.element_size() for r in rows]
    offs, o = [], 0
    for sz in sizes:
        offs.append(o)
        o += (sz + 255) // 256 * 256
    t, root = pool.take(o)
    for r, off, sz in zip(rows, offs, sizes):
        if n:
            t[off:off + sz].view(r.dtype).copy_(r[:n], non_blocking=True)
    (stream or torch.cuda.current_stream()).synchronize()
    np_dt = {torch.int64: np.int64, torch.int16: np.int16, torch.int8: np.int8, torch.int32: np.int32,
             torch.float32: np.float32, torch.uint8: np.uint8}
    return [root[off:off + sz].view(np_dt[r.dtype]) for r, off, sz in zip(rows, offs, sizes)]


def d2h_segments(pool: PinnedPool, counts, rows2d, stream=None, sync: bool = True):
    """Device [nseg][cap] output pools -> host: the first counts[g] elements of
    every segment, packed per row into one pinned block (async copies, one
    synchronize).  Returns, per row, a list of per-segment numpy views."""
    import torch

    counts = [int(c) for c in counts]
    total = sum(counts)
    offs, o = [], 0
    for r in rows2d:
        offs.append(o)
        o += (total * r.element_size() + 255) // 256 * 256
    t, root = pool.take(max(o, 1))
    np_dt = {torch.int64: np.int64, torch.int16: np.int16, torch.int8: np.int8}
    out = []
    for r, base in zip(rows2d, offs):
        es = r.element_size()
        views, e = [], 0
        for g, n in enumerate(counts):
            if n:
                t[base + e * es:base + (e + n) * es].view(r.dtype).copy_(r[g, :n], non_blocking=True)
            views.append(root[base + e * es:base + (e + n) * es].view(np_dt[r.dtype]))
            e += n
        out.append(views)
    if sync:
        (stream or torch.cuda.current_stream()).synchronize()
    return out


def compact_launch(counts_dev, rows2d, scratch: dict) -> bool:
    """Enqueue evs_compact_segments of an evs_step output's four SoA rows into
    the device staging arrays of ``scratch`` on the current stream (no host
    round trip: the counts stay on the device).  False when ``scratch`` has no
    staging yet (the first window sizes it, see d2h_packed)."""
    n = scratch.get("n", 0)
    if not n:
        return False
    L = _lib.load()
    rc = L.evs_compact_segments(counts_dev.shape[0], counts_dev.data_ptr(), rows2d[0].shape[1],
                                *[r.data_ptr() for r in rows2d], *[b.data_ptr() for b in scratch["bufs"]], n,
                                _lib.stream_ptr())
    _lib.check(rc, "evs_compact_segments")
    return True


def d2h_packed(pool: PinnedPool, counts_host, rows2d, scratch: dict, compacted: bool, sync: bool = True):
    """Device -> pinned host copy of an evs_step output's four SoA rows.  When
    compact_launch packed the segments and they fit, each row crosses PCIe in
    ONE copy (measured 44 -> 52 GB/s next to H2D traffic); otherwise per
    segment (d2h_segments), and the staging grows for the next window.
    Returns, per row, a list of per-segment numpy views."""
    import torch

    counts = [int(c) for c in counts_host]
    total = sum(counts)
    if not compacted or total > scratch.get("n", 0):
        if total > scratch.get("n", 0):  # grow with headroom (allocation synchronises: rare)
            n = max(1 << (total + total // 4).bit_length(), 1 << 16)
            # the old staging may still be written by an in-flight compaction: keep it alive
            scratch.setdefault("retired", []).append(scratch.get("bufs"))
            scratch.update(n=n, bufs=[torch.empty(n, dtype=r.dtype, device=r.device) for r in rows2d])
        return d2h_segments(pool, counts, rows2d, sync=sync)
    offs, o = [], 0
    for r in rows2d:
        offs.append(o)
        o += (total * r.element_size() + 255) // 256 * 256
    t, root = pool.take(max(o, 1))
    np_dt = {torch.int64: np.int64, torch.int16: np.int16, torch.int8: np.int8}
    out = []
    for r, b, base in zip(rows2d, scratch["bufs"], offs):
        es = r.element_size()
        if total:
            t[base:base + total * es].view(r.dtype).copy_(b[:total], non_blocking=True)
        views, e = [], 0
        for n in counts:
            views.append(root[base + e * es:base + (e + n) * es].view(np_dt[r.dtype]))
            e += n
        out.append(views)
    if sync:
        torch.cuda.current_stream().synchronize()
    return out


def upload_frame(values, device, staging_cache: dict | None = None):
    """Host numpy (H, W) float32 -> device tensor.  A direct copy from the
    caller's pageable array (the driver stages it) measured faster than an
    extra memcpy into a pinned buffer; ``staging_cache`` is kept for callers."""
    import torch

    if type(values).__module__.startswith("torch"):
        return values.to(device=device, dtype=torch.float32).contiguous()
    arr = np.ascontiguousarray(values, np.float32)
    return torch.from_numpy(arr).to(device)
