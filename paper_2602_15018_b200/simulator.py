"""Batched, device-resident event simulator (the production path).

``EventSimulator`` steps S independent event cameras ("streams") together,
T frames per call, with every per-pixel state and every output buffer in
HBM.  One call = one ``evs_step`` (validation prologue, fused generate,
column scan, ordering pass) for all S x T (stream, frame) segments; optional
exact noise is generated per segment and merged into the canonical order;
optional representations (signed-polarity histogram per window,
accumulate_events_to_image semantics; B-bin voxel grid) are accumulated on
the device.  ``capture()``/``replay()`` run whole frame sequences as one CUDA
graph with the step clock advancing on the device.

This is the batched counterpart of the reference's per-tick event block in
``SimNode.step_once`` (orchestrator.py:159-172): generate -> (noise, seeded
``_mix64(seed, 0x6E6F6973, k)``) -> concat -> canonical_sort.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .events.model import init_pixel_states
from .events.types import DeviceEventBatch, EventCameraConfig, IntensityFrame
from .runtime import StepEngine, StepShape


def mix64(*parts: int) -> int:
    """orchestrator.py:51-56: FNV-style seed mixing used for per-tick noise seeds."""
    h = 0xCBF29CE484222325
    for p in parts:
        h ^= p & 0xFFFFFFFFFFFFFFFF
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


@dataclass
class StepResult:
    """Device-resident outputs of one step (views into the engine's pools)."""

    sim: "EventSimulator"
    counts: np.ndarray       # [S, T] events written per segment
    dropped: np.ndarray      # [S, T]
    reservations: np.ndarray  # [S, T]

    def segment(self, s: int, f: int = 0) -> DeviceEventBatch:
        return self.sim.segment(s, f)


class EventSimulator:
    def __init__(self, width: int, height: int, streams: int = 1, frames_per_step: int = 1,
                 config: EventCameraConfig | None = None, tick_us: int = 1000, canonical: bool = True,
                 device=None):
        import torch

        _lib.require_cuda()
        self.W, self.H, self.S, self.T = int(width), int(height), int(streams), int(frames_per_step)
        self.P = self.W * self.H
        self.cfg = config or EventCameraConfig()
        self.tick = int(tick_us)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.canonical = canonical
        self.cap = int(self.cfg.capacity(self.W, self.H))
        self.ref = torch.empty((self.S, self.H, self.W), dtype=torch.float32, device=self.device)
        self.last = torch.empty((self.S, self.H, self.W), dtype=torch.int64, device=self.device)
        self.thp = torch.empty_like(self.ref)
        self.thn = torch.empty_like(self.ref)
        self.uniform = None
        self.engine: StepEngine | None = None
        self.t_next = 0
        self.step_index = 0
        self._noise_seed = None
        self._last_noise = None

    # -- construction (init_pixel_states per stream, model.py:42-67) ----------
    def reset(self, frames0, seeds=None, t0: int = 0) -> None:
        """Initialise every stream from its first frame (host numpy, exact thresholds)."""
        seeds = list(range(self.S)) if seeds is None else list(seeds)
        uni = []
        for s in range(self.S):
            f0 = frames0[s]
            f0 = f0.detach().cpu().numpy() if type(f0).__module__.startswith("torch") else np.asarray(f0)
            st = init_pixel_states(IntensityFrame(self.W, self.H, t0, f0), self.cfg, seed=seeds[s])
            self.ref[s].copy_(st.d_ref_log)
            self.last[s].copy_(st.d_last_event_t)
            self.thp[s].copy_(st.d_thresholds_pos)
            self.thn[s].copy_(st.d_thresholds_neg)
            uni.append(st.uniform_thresholds)
        self.uniform = uni[0] if all(u == uni[0] and u is not None for u in uni) else None
        shape = StepShape(self.S, self.T, self.H, self.W, self.cap,
                          _lib.EVS_ORDER_CANONICAL if self.canonical else _lib.EVS_ORDER_PIXEL_MAJOR,
                          self.tick, float(self.cfg.log_eps), int(self.cfg.refractory_us), self.uniform)
        self.engine = StepEngine(shape, self.device)
        self.t_next = int(t0)
        self.step_index = 0

    # -- stepping --------------------------------------------------------------
    def _check_frames(self, frames, device: bool = True):
        """The kernels read S*T*H*W float32 values through a raw pointer: reject
        anything else before launching.  Returns the [S, T, H, W] view."""
        import torch

        full = (self.S, self.T, self.H, self.W)
        if device:
            if not isinstance(frames, torch.Tensor):
                raise TypeError("frames must be a CUDA float32 tensor (use step_host for host arrays)")
            if frames.dtype != torch.float32:
                raise ValueError(f"frames must be float32, got {frames.dtype}")
            if frames.device != self.device:
                raise ValueError(f"frames must be on {self.device}, got {frames.device}")
            if not frames.is_contiguous():
                raise ValueError("frames must be contiguous")
        shape = tuple(frames.shape)
        if shape == (self.S, self.H, self.W) and self.T == 1:
            return frames.unsqueeze(1) if device else frames[:, None]
        if shape != full:
            raise ValueError(f"frames shape {shape} != (streams, frames_per_step, height, width) = {full}"
                             + (" (or (streams, height, width) when frames_per_step == 1)" if self.T == 1 else ""))
        return frames

    def step(self, frames, validate: bool = True, sync: bool = False, stage_events=None):
        """Advance every stream by T frames.  frames: contiguous float32 CUDA tensor
        [S, T, H, W] on this simulator's device (or [S, H, W] when T == 1).
        Asynchronous unless sync=True."""
        eng = self.engine
        assert eng is not None, "call reset() first"
        frames = self._check_frames(frames)
        eng.launch(frames, self.ref, self.last, self.thp, self.thn, t0=self.t_next, tick=self.tick,
                   validate=validate, stage_events=stage_events)
        self.t_next += self.T * self.tick
        self.step_index += 1
        if sync:
            return self.result()
        return None

    def result(self) -> StepResult:
        counts, dropped, res, bad = self.engine.fetch_info()
        if bad != _lib.NO_BAD:
            self.engine.reset_bad()
            s, rem = divmod(int(bad), self.T * self.P)
            f, pix = divmod(rem, self.P)
            y, x = divmod(pix, self.W)
            raise ValueError(f"invalid intensity at stream {s}, frame {f}, pixel (x={x}, y={y})")
        sh = (self.S, self.T)
        return StepResult(self, counts.reshape(sh), dropped.reshape(sh), res.reshape(sh))

    def segment(self, s: int, f: int = 0) -> DeviceEventBatch:
        """Events of stream s, frame f of the last step (canonical order), on the device."""
        g = s * self.T + f
        n = int(self.engine.info[0, g].item())
        e = self.engine
        return DeviceEventBatch(e.ev_t[g, :n], e.ev_x[g, :n], e.ev_y[g, :n], e.ev_p[g, :n],
                                dropped_count=int(e.info[1, g].item()), canonical=self.canonical)

    def step_host(self, frames_host, validate: bool = True):
        """Host-buffer counterpart of step(): frames_host is a float32 numpy array
        [S, T, H, W] (or [S, H, W] when T == 1); returns the events of every
        (stream, frame) as host EventBatch objects, list [S][T], canonical order.
        The result arrays are views into reusable pinned blocks (valid while held)."""
        import torch

        from .events.types import EventBatch
        from .runtime import PinnedPool, compact_launch, d2h_packed

        fr = self._check_frames(np.ascontiguousarray(frames_host, np.float32), device=False)
        dfr = torch.from_numpy(fr).to(self.device)
        self.step(dfr, validate=validate)
        e = self.engine
        rows = [e.ev_t, e.ev_x, e.ev_y, e.ev_p]
        if not hasattr(self, "_pool"):
            self._pool = PinnedPool()
        if not hasattr(self, "_step_scratch"):
            self._step_scratch = {}
        packed = compact_launch(e.info[0], rows, self._step_scratch)  # behind the step, before the host read
        res = self.result()
        t, x, y, p = d2h_packed(self._pool, res.counts.ravel(), rows, self._step_scratch, packed)
        out = []
        for s in range(self.S):
            row = []
            for f in range(self.T):
                g = s * self.T + f
                row.append(EventBatch(t=t[g].view(np.uint64), x=x[g].view(np.uint16), y=y[g].view(np.uint16),
                                      polarity=p[g], dropped_count=int(res.dropped[s, f]),
                                      canonical=self.canonical))
            out.append(row)
        return out

    def run_host(self, windows, validate: bool = True):
        """Pipelined host-buffer stepping: for each float32 numpy window
        [S, T, H, W] of ``windows`` (ideally page-locked, see ``pin_host``)
        yield the host EventBatch list [S][T] of that window, in order.

        Window i+1's host->device copy and window i's device->host copy run on
        their own streams while window i+1 computes; two output pools (two
        engines sharing this simulator's state) let a window's results drain
        while the next one is generated.  Results are views into pinned blocks
        (valid while held).
        """
        import torch

        from .events.types import EventBatch
        from .runtime import PinnedPool, StepEngine, compact_launch, d2h_packed

        assert self.engine is not None, "call reset() first"
        dev = self.device
        comp = torch.cuda.current_stream(dev)
        h2d = torch.cuda.Stream(dev)
        d2h = torch.cuda.Stream(dev)
        if not hasattr(self, "_pool"):
            self._pool = PinnedPool()
        if not hasattr(self, "_engine2"):
            self._engine2 = StepEngine(self.engine.shape, dev)
        engines = [self.engine, self._engine2]
        fbuf = [torch.empty((self.S, self.T, self.H, self.W), dtype=torch.float32, device=dev) for _ in range(2)]
        ev_h2d = [torch.cuda.Event() for _ in range(2)]
        ev_comp = [torch.cuda.Event() for _ in range(2)]
        ev_d2h = [torch.cuda.Event() for _ in range(2)]
        if not hasattr(self, "_rh_scratch"):  # device staging of the packed segments, one per pool
            self._rh_scratch = [{}, {}]       # (kept across calls: allocating it synchronises)
        scratch = self._rh_scratch
        for e in ev_comp + ev_d2h:
            e.record(comp)

        def upload(i, win):
            fr = self._check_frames(np.ascontiguousarray(win, np.float32), device=False)
            with torch.cuda.stream(h2d):
                h2d.wait_event(ev_comp[i % 2])  # window i-2 has finished reading this buffer
                fbuf[i % 2].copy_(torch.from_numpy(fr), non_blocking=True)
                ev_h2d[i % 2].record(h2d)

        it = iter(windows)
        win = next(it, None)
        if win is None:
            return
        upload(0, win)
        pending = None  # (batches, copy-done event) of the previous window
        i = 0
        while True:
            eng = engines[i % 2]
            comp.wait_event(ev_h2d[i % 2])
            comp.wait_event(ev_d2h[i % 2])  # window i-2's results have left this pool
            eng.launch(fbuf[i % 2], self.ref, self.last, self.thp, self.thn, t0=self.t_next, tick=self.tick,
                       validate=validate, stream=comp)
            rows = [eng.ev_t, eng.ev_x, eng.ev_y, eng.ev_p]
            with torch.cuda.stream(comp):  # pack the segments behind the step (copy engine stays busy)
                packed = compact_launch(eng.info[0], rows, scratch[i % 2])
            ev_comp[i % 2].record(comp)
            self.t_next += self.T * self.tick
            self.step_index += 1
            win = next(it, None)
            if win is not None:
                upload(i + 1, win)  # overlaps window i's compute and window i-1's drain
            counts, dropped, res, bad = eng.fetch_info()  # waits for window i's compute
            if bad != _lib.NO_BAD:
                eng.reset_bad()
                raise ValueError(f"invalid intensity in window {i} (flat index {int(bad)})")
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_comp[i % 2])
                t, x, y, p = d2h_packed(self._pool, counts, rows, scratch[i % 2], packed, sync=False)
                ev_d2h[i % 2].record(d2h)
            dr = dropped.reshape(self.S, self.T)
            batches = [[EventBatch(t=t[g].view(np.uint64), x=x[g].view(np.uint16), y=y[g].view(np.uint16),
                                   polarity=p[g], dropped_count=int(dr[g // self.T, g % self.T]),
                                   canonical=self.canonical)
                        for g in range(s * self.T, (s + 1) * self.T)] for s in range(self.S)]
            if pending is not None:
                pending[1].synchronize()
                yield pending[0]
            pending = (batches, ev_d2h[i % 2])
            if win is None:
                pending[1].synchronize()
                yield pending[0]
                return
            i += 1

    @staticmethod
    def pin_host(array: np.ndarray) -> np.ndarray:
        """Page-lock a host numpy array in place (cudaHostRegister) so copies from
        it run at full PCIe rate; returns the array.  Unpin with unpin_host."""
        import torch

        rc = torch.cuda.cudart().cudaHostRegister(array.ctypes.data, array.nbytes, 0)
        if int(rc) != 0:
            raise RuntimeError(f"cudaHostRegister failed ({int(rc)})")
        return array

    @staticmethod
    def unpin_host(array: np.ndarray) -> None:
        import torch

        torch.cuda.cudart().cudaHostUnregister(array.ctypes.data)

    # -- CUDA graph replay -------------------------------------------------------
    def capture(self, frame_windows) -> None:
        """Capture one graph stepping through `frame_windows` ([S, T, H, W] each) in order."""
        frame_windows = [self._check_frames(w) for w in frame_windows]
        self.engine.capture(frame_windows, self.ref, self.last, self.thp, self.thn, tick=self.tick,
                            t0=self.t_next)
        self._graph_len = len(frame_windows)

    def replay(self) -> None:
        self.engine.replay()
        self.t_next += self._graph_len * self.T * self.tick
        self.step_index += self._graph_len

    # -- noise + representations --------------------------------------------------
    def segment_with_noise(self, s: int, f: int, seed: int) -> DeviceEventBatch:
        """Signal events of (s, f) merged with exact noise seeded like SimNode
        (orchestrator.py:167-171), canonical order."""
        from .noise import noise_params, run_noise
        from .represent import merge_canonical

        sig = self.segment(s, f)
        if self.cfg.noise_rate_hz <= 0:
            return sig
        t_now = self.t_next - (self.T - 1 - f) * self.tick
        t_prev = t_now - self.tick
        p = noise_params(self.W, self.H, t_prev, t_now, self.cfg.noise_rate_hz, seed, order=0)
        n, b = run_noise(p, self.device)
        noise = DeviceEventBatch(b["t"][:n], b["x"][:n], b["y"][:n], b["p"][:n], 0, False)
        from .represent import canonical_sort

        return merge_canonical(sig, canonical_sort(noise))

    def histogram(self, batch: DeviceEventBatch, window_us: int, t_end: int):
        from .represent import accumulate

        return accumulate(batch, window_us, t_end, self.W, self.H, device_output=True)

    def voxel_window(self, s: int = 0, bins: int = 5, noise_seeds=None, _noise_capacity=None):
        """B-bin voxel grid, f32 (bins, H, W) on the device, of
        stream s over the last step's window [t_next - T*tick, t_next): the
        signal events of its T frames plus, when config.noise_rate_hz > 0 and
        ``noise_seeds`` (one per frame) is given, the exact noise of every
        frame (inject_noise_events, model.py:174-212, seeded per tick as
        SimNode does, orchestrator.py:167-171).  The voxel sum is order
        independent (exact int64 numerators, one rounding), so nothing is
        sorted or merged: the signal numerators come straight from the step's
        per-tile key regions (evs_step_voxel: one CTA per tile, shared-memory
        accumulation), one batched noise
        launch set (evs_noise_batch) fills a pooled buffer with the T frames'
        noise, one segmented accumulation adds it, one
        rounding, and one host read per window (the noise kernels' retry
        flags; a flagged frame is redone by the retrying path)."""
        import ctypes

        import torch

        from .noise import noise_params, run_noise

        L = _lib.load()
        e = self.engine
        assert e is not None, "call reset() first"
        T, W, H, P = self.T, self.W, self.H, self.P
        t1 = self.t_next
        t0 = t1 - T * self.tick
        nbytes = int(L.evs_voxel_workspace_bytes(bins, W, H))
        ws = getattr(self, "_vox_ws", None)
        if ws is None or ws.numel() < nbytes:
            ws = self._vox_ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        out = torch.empty((bins, H, W), dtype=torch.float32, device=self.device)
        st = _lib.stream_ptr()
        use_noise = self.cfg.noise_rate_hz > 0 and noise_seeds is not None
        g0 = s * T

        def vox(nseg, counts, cstride, sstride, t, x, y, p, flags):
            rc = L.evs_voxel_segments(nseg, counts, cstride, sstride, t, x, y, p, t0, t1, bins, W, H, flags,
                                      out.data_ptr(), ws.data_ptr(), ws.numel(), st)
            _lib.check(rc, "evs_voxel_segments")

        def signal(flags):
            # from the step's per-tile regions (shared-memory accumulation, every pixel written)
            fin = flags & _lib.EVS_VOXEL_FINALIZE
            rc = L.evs_step_voxel(ctypes.byref(e.params), ctypes.byref(e.bufs), e.workspace.data_ptr(),
                                  e.workspace.numel(), s, t0, t1, bins, fin, out.data_ptr(), ws.data_ptr(),
                                  ws.numel(), st)
            _lib.check(rc, "evs_step_voxel")

        signal(0 if use_noise else _lib.EVS_VOXEL_FINALIZE)
        if not use_noise:
            return out
        seeds = list(noise_seeds)
        if len(seeds) != T:
            raise ValueError(f"need {T} noise seeds (one per frame), got {len(seeds)}")
        params = [noise_params(W, H, t0 + f * self.tick, t0 + (f + 1) * self.tick, self.cfg.noise_rate_hz,
                               seeds[f], order=0) for f in range(T)]
        if params[0].lam <= 0:
            vox(0, None, 1, 0, None, None, None, None, _lib.EVS_VOXEL_FINALIZE)
            return out
        cap = max(int(L.evs_noise_capacity(ctypes.byref(p))) for p in params)
        if _noise_capacity is not None:
            cap = int(_noise_capacity)
        for p in params:
            p.capacity = cap
        parr = (_lib.NoiseParams * T)(*params)
        nws = int(L.evs_noise_batch_workspace_bytes(parr, T))
        pool = getattr(self, "_noise_pool", None)
        if pool is None or pool["t"].shape[0] < T or pool["t"].shape[1] < cap or pool["ws"].numel() < nws:
            pool = self._noise_pool = {
                "t": torch.empty((T, cap), dtype=torch.int64, device=self.device),
                "x": torch.empty((T, cap), dtype=torch.int16, device=self.device),
                "y": torch.empty((T, cap), dtype=torch.int16, device=self.device),
                "p": torch.empty((T, cap), dtype=torch.int8, device=self.device),
                "meta": torch.zeros((T, 4), dtype=torch.int64, device=self.device),
                "ws": torch.empty(max(nws, 1), dtype=torch.uint8, device=self.device)}
        nt, nx, ny, npol, meta, nw = (pool[k] for k in ("t", "x", "y", "p", "meta", "ws"))
        stride = nt.shape[1]
        rc = L.evs_noise_batch(parr, T, nt.data_ptr(), nx.data_ptr(), ny.data_ptr(), npol.data_ptr(), stride,
                               meta.data_ptr(), nw.data_ptr(), nw.numel(), st)
        _lib.check(rc, "evs_noise_batch")
        vox(T, meta[:, 1].data_ptr(), 4, stride, nt.data_ptr(), nx.data_ptr(), ny.data_ptr(), npol.data_ptr(),
            _lib.EVS_VOXEL_FINALIZE)
        retry = meta[:T, 2:4].cpu().numpy()
        if not retry.any():
            return out
        # rare: a frame's draw range or capacity was short -- redo the window with
        # the retrying per-frame path (same result, noise_params rebuilt fresh)
        signal(0)
        for f in range(T):
            p = noise_params(W, H, t0 + f * self.tick, t0 + (f + 1) * self.tick, self.cfg.noise_rate_hz,
                             seeds[f], order=0)
            n, b = run_noise(p, self.device)
            cnt = torch.tensor([n], dtype=torch.int64, device=self.device)
            vox(1, cnt.data_ptr(), 1, 0, b["t"].data_ptr(), b["x"].data_ptr(), b["y"].data_ptr(),
                b["p"].data_ptr(), 0)
        vox(0, None, 1, 0, None, None, None, None, _lib.EVS_VOXEL_FINALIZE)
        return out

    def histograms(self, window_us: int, t_end: int | None = None):
        """accumulate_events_to_image (model.py:249-262) of every stream's events
        of the last step with t in [t_end - window_us, t_end) (default t_end: the
        end of the step): int64 [S, H, W] on the device, one launch for all
        streams (evs_step_histogram)."""
        import ctypes

        import torch

        e = self.engine
        assert e is not None, "call reset() first"
        if window_us <= 0:
            raise ValueError("window_us must be positive")
        t_end = self.t_next if t_end is None else int(t_end)
        out = torch.empty((self.S, self.H, self.W), dtype=torch.int64, device=self.device)
        L = _lib.load()
        rc = L.evs_step_histogram(ctypes.byref(e.params), ctypes.byref(e.bufs), e.workspace.data_ptr(),
                                  e.workspace.numel(), int(window_us), t_end, out.data_ptr(), _lib.stream_ptr())
        _lib.check(rc, "evs_step_histogram")
        return out

    def voxel(self, batch: DeviceEventBatch, t0: int, t1: int, bins: int = 5):
        from .represent import voxel_grid

        return voxel_grid(batch, t0, t1, self.W, self.H, bins=bins, device_output=True)
