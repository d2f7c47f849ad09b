#!/usr/bin/env python
"""Benchmark of the B200 event-camera hot path (one JSON line on rank 0).

Headline (default, BASELINE.json configs[1]): HD 1280x720 camera, C=0.15,
refractory 100 us, 1000 us ticks, synthetic moving texture
(events_bench.py:19-26), time-ordered (t, x, y, p) output per frame.  A
"step" is one evs_step over T consecutive frames of the camera (default
T=50; every frame still gets its own canonical event segment), replayed as a
CUDA graph with the step clock on the device.  Frames cycle through a
pre-uploaded ring of lcm(T, 50) frames (>= 184 MB > 126 MB L2), so every step
reads its frames from HBM.  The same workload at one frame per launch (the
reference's per-frame call granularity) is reported in "per_frame_launch".
After the timed region the same launch shape is checked against an oracle
fixture ("self_check"); a mismatch fails the run.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--frames-per-step T] [--config 2|1|3|4|5]
  python bench.py --impl reference ...   # the reference's own CPU path on the host cores

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one process per GPU, NCCL); under torchrun WORLD_SIZE must equal N.

Other BASELINE configs (--config):
  1  DAVIS 346x260, C=0.2, capacity 32 P, one stream per rank (T=50)
  3  64 independent 640x480 cameras sharded over the ranks (s -> floor(s N / 64), T=10)
  4  1920x1080, C=0.05, exact 10 Hz noise, 5-bin voxel grid per 20-frame window, one camera per rank
  5  256 DAVIS streams sharded over the ranks (T=4), per-stream event histograms of every step
     window, and the step's events gathered to rank 0 as packed 4-byte keys over NCCL
Configs 2, 1 and 4 are replicas (weak scaling: one camera per rank); 3 and 5
shard a fixed stream set (strong scaling).  value = units of all ranks /
max-over-ranks device time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W, H = 1280, 720
C_TH = 0.15
REFR = 100
TICK = 1000
DRIFT = 0.02
METRIC = "simulated HD (1280x720) frames/s and Mevents/s per GPU; % of HBM roofline"
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

# BASELINE.json configs -> workloads (stream phase 0.137 s, state seed s)
CONFIGS = {
    "2": dict(W=1280, H=720, C=0.15, refr=100, T=50, cap_px=8, streams=None, noise=0.0,
              metric=METRIC, unit="frames/s",
              workload="HD 1280x720 single camera per GPU, C=0.15, refractory 100us, 1000us ticks, moving texture, "
                       "canonical (t,y,x,p) output per frame"),
    "1": dict(W=346, H=260, C=0.2, refr=0, T=50, cap_px=32, streams=None, noise=0.0,
              metric="DAVIS 346x260 frames/s (1000 synthetic moving-texture frames per stream), C=0.2; % of HBM roofline",
              unit="frames/s",
              workload="DAVIS 346x260 single stream per GPU, C=0.2, capacity 32P (events_bench.py:40), moving texture"),
    "3": dict(W=640, H=480, C=0.2, refr=0, T=10, cap_px=8, streams=64, noise=0.0,
              metric="640x480 camera-frames/s over 64 independent cameras; % of HBM roofline", unit="camera-frames/s",
              workload="64 independent 640x480 cameras (s -> rank floor(s*N/64)), C=0.2, moving texture"),
    "4": dict(W=1920, H=1080, C=0.05, refr=0, T=20, cap_px=8, streams=None, noise=10.0,
              metric="1920x1080 frames/s with exact 10 Hz noise and a 5-bin voxel grid per 20-frame window",
              unit="frames/s",
              workload="1920x1080 single camera per GPU, C=0.05 (multi-crossing), exact 10 Hz noise per frame, "
                       "5-bin voxel grid per 20-frame window"),
    "5": dict(W=346, H=260, C=0.2, refr=0, T=4, cap_px=8, streams=256, noise=0.0,
              metric="346x260 stream-frames/s over 256 streams + per-stream event histograms + NCCL gather of the "
                     "events to rank 0", unit="stream-frames/s",
              workload="256 DAVIS 346x260 streams (s -> rank floor(s*N/256)), C=0.2, per-stream signed histogram "
                       "of every step window, events gathered to rank 0 as packed 4-byte keys"),
}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    def __init__(self, index: int):
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # pragma: no cover - no NVML
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(P, A, E, refr, uniform=True, T=1, S=1):
    """SURVEY.md 8(d), summed over S streams: 4PT + 4P + 12A_T + 8A_T[refr] + 8P[non-uniform] + 13E
    (A = pixels whose state changed over the call, all streams; E = events written, all segments)."""
    return S * (4 * P * T + 4 * P + (0 if uniform else 8 * P)) + 12 * A + (8 * A if refr > 0 else 0) + 13 * E


def config_dict(cfg, T, world, sharded):
    d = {"workload": cfg["workload"], "frames_per_step": T, "capacity_per_frame": cfg["cap_px"] * cfg["W"] * cfg["H"],
         "l2": "inputs cycle through a frame ring larger than the 126 MB L2"}
    if sharded:
        d["streams"] = cfg["streams"]
        d["parallelism"] = f"streams sharded over {world} GPU(s)"
    else:
        d["parallelism"] = f"replicas x{world}" if world > 1 else "single GPU"
    return d


# --------------------------------------------------------------------------- inputs
def device_texture_ring(width, height, frames, drift, phase0, dev):
    """Ring of `frames` frames on the device, frame k = _texture_frame(phase0 + (k mod 50) * drift)
    (events_bench.py:19-26, computed on the host in f64 like the reference, uploaded once)."""
    import torch

    from paper_2602_15018_b200.synth import PERIOD_FRAMES, texture_frame

    base = [torch.from_numpy(texture_frame(width, height, phase0 + k * drift)).to(dev)
            for k in range(min(frames, PERIOD_FRAMES))]
    out = torch.empty((frames, height, width), dtype=torch.float32, device=dev)
    for k in range(frames):
        out[k].copy_(base[k % PERIOD_FRAMES])
    return out


def gpu_texture_windows(width, height, phases, T, dev):
    """[lcm(T, 50) / T windows][S][T][H][W] moving-texture frames of S streams
    evaluated on the GPU in f64 (multi-stream throughput inputs; the 50-frame
    period of the texture lines up with the windows, so cycling never jumps)."""
    import torch

    n = T * 50 // math.gcd(T, 50)
    x = torch.arange(width, dtype=torch.float64, device=dev) / width
    y = torch.arange(height, dtype=torch.float64, device=dev) / height
    grid = y[:, None] * 2.0 + x[None, :] * 3.0
    out = torch.empty((n // T, len(phases), T, height, width), dtype=torch.float32, device=dev)
    for s, ph in enumerate(phases):
        for k in range(n):
            out[k // T, s, k % T] = (0.5 + 0.45 * torch.sin(2.0 * math.pi * (grid + (ph + ((k + 1) % 50) * DRIFT)))
                                     ).float()
    return out


# --------------------------------------------------------------------------- self-check (config 2)
FIXTURE = os.path.join(ROOT, "tests", "golden", "bench_hd_t50.json")


def _sha1(arrays) -> str:
    import hashlib

    h = hashlib.sha1()
    for a, dt in zip(arrays, (np.uint64, np.uint16, np.uint16, np.int8)):
        h.update(np.ascontiguousarray(np.asarray(a).astype(dt, copy=False)).tobytes())
    return h.hexdigest()


def verify_launch_shape(dev, T: int, frames: int = 150, pipelined: bool = False):
    """Self-check of the benchmarked launch shape (HD, T frames per evs_step,
    capacity 8P, fused validation, CUDA-graph replay with the device clock)
    against the oracle fixture tests/golden/bench_hd_t50.json (per-frame
    counts, drops, reservations, SHA-1 of the canonical events; the state).
    The first step runs eagerly, the following ones as graph replays, exactly
    like the timed region (pipelined: the replays alternate two engines on two
    streams, runtime.PipelinedSteps).  Returns the list of mismatching frames."""
    import torch

    from paper_2602_15018_b200 import _lib
    from paper_2602_15018_b200 import events as ev
    from paper_2602_15018_b200.runtime import StepEngine, StepShape
    from paper_2602_15018_b200.synth import PERIOD_FRAMES, texture_frame

    with open(FIXTURE) as f:
        fx = json.load(f)
    frames = min(frames, len(fx["frames"]))
    P = W * H
    cfg = ev.EventCameraConfig(c_pos=C_TH, c_neg=C_TH, refractory_us=REFR)
    ring_len = T * PERIOD_FRAMES // math.gcd(T, PERIOD_FRAMES)
    ring = device_texture_ring(W, H, ring_len, DRIFT, 0.0, dev)
    st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, 0.0)), cfg, seed=0)
    eng = StepEngine(StepShape(1, T, H, W, 8 * P, _lib.EVS_ORDER_CANONICAL, TICK, cfg.log_eps, REFR,
                               st.uniform_thresholds), dev)
    nsteps = (frames + T - 1) // T
    bad = []

    def check(e, i):
        counts, dropped, res, badpx = e.fetch_info()
        if badpx != _lib.NO_BAD:
            bad.append(f"invalid frame in step {i}")
            return
        for f in range(T):
            j = i * T + f
            if j >= frames:
                break
            n = int(counts[f])
            got = {"count": n, "dropped": int(dropped[f]), "reservations": int(res[f]),
                   "sha1": _sha1([e.ev_t[f, :n].cpu().numpy(), e.ev_x[f, :n].cpu().numpy(),
                                  e.ev_y[f, :n].cpu().numpy(), e.ev_p[f, :n].cpu().numpy()])}
            if got != fx["frames"][j]:
                bad.append(j)

    win0 = ring[0:T]
    eng.launch(win0, st.d_ref_log, st.d_last_event_t, t0=0, tick=TICK, validate=True)
    torch.cuda.synchronize()
    check(eng, 0)
    if pipelined and nsteps >= 3:
        from paper_2602_15018_b200.runtime import PipelinedSteps

        pipe = PipelinedSteps(eng.shape, dev)
        pipe.engines[0] = eng
        i = 1
        while i < nsteps:
            wins = [ring[((i + j) * T) % ring_len:((i + j) * T) % ring_len + T] for j in range(2)]
            pipe.capture(wins, st.d_ref_log, st.d_last_event_t, tick=TICK, t0=i * T * TICK)
            pipe.replay()
            torch.cuda.synchronize()
            for j in range(2):
                if i + j < nsteps:
                    check(pipe.engines[j], i + j)
            i += 2
    for i in range(1, nsteps if not (pipelined and nsteps >= 3) else 1):
        win = ring[(i * T) % ring_len:(i * T) % ring_len + T]
        if i == 1 or (T % PERIOD_FRAMES):  # (windows repeat when T is a multiple of the period)
            eng.capture([win], st.d_ref_log, st.d_last_event_t, tick=TICK, t0=i * T * TICK)
        eng.replay()
        torch.cuda.synchronize()
        check(eng, i)
    if nsteps * T == frames == len(fx["frames"]):
        import hashlib

        h = hashlib.sha1()
        h.update(st.d_ref_log.cpu().numpy().tobytes())
        h.update(st.d_last_event_t.cpu().numpy().tobytes())
        if h.hexdigest() != fx["state_sha1"]:
            bad.append("state")
    return bad


def measure_t1(args, dev, cfg, phase0, rank, order=None):
    """The same workload with one frame per evs_step (the reference's per-frame
    call granularity), graph-replayed: (a) consecutive steps overlapped on two
    streams (runtime.PipelinedSteps: step k+1's K1 runs while step k's
    ordering finishes) -- the frame rate; (b) strictly one step after the other
    -- the latency of one frame.  order: canonical (default) or pixel-major
    (generate_events_serial order, model.py:140)."""
    import torch

    from paper_2602_15018_b200 import _lib
    from paper_2602_15018_b200 import events as ev
    from paper_2602_15018_b200.runtime import PipelinedSteps, StepEngine, StepShape
    from paper_2602_15018_b200.synth import PERIOD_FRAMES, texture_frame

    P = W * H
    ring = device_texture_ring(W, H, PERIOD_FRAMES, DRIFT, phase0, dev)
    order = _lib.EVS_ORDER_CANONICAL if order is None else order
    reps = max(2, args.steps // PERIOD_FRAMES)
    out = {}
    for mode in ("pipelined", "serial"):
        st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, phase0)), cfg, seed=rank)
        shape = StepShape(1, 1, H, W, 8 * P, order, TICK, cfg.log_eps, REFR, st.uniform_thresholds)
        runner = PipelinedSteps(shape, dev) if mode == "pipelined" else StepEngine(shape, dev)
        eng0 = runner.engines[0] if mode == "pipelined" else runner
        for k in range(5):
            eng0.launch(ring[k:k + 1], st.d_ref_log, st.d_last_event_t, t0=k * TICK, tick=TICK)
        if mode == "pipelined":
            for k in range(5, 7):  # (kernel attributes of the second engine)
                runner.engines[1].launch(ring[k:k + 1], st.d_ref_log, st.d_last_event_t, t0=k * TICK, tick=TICK)
        k0 = 7 if mode == "pipelined" else 5
        runner.capture([ring[(k0 + i) % PERIOD_FRAMES:(k0 + i) % PERIOD_FRAMES + 1] for i in range(PERIOD_FRAMES)],
                       st.d_ref_log, st.d_last_event_t, tick=TICK, t0=k0 * TICK)
        runner.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            runner.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        frames = reps * PERIOD_FRAMES
        out[mode] = {"frames_per_s": frames / (ms / 1e3), "us_per_frame": 1e3 * ms / frames, "frames": frames}
    res = dict(out["pipelined"])
    res["mode"] = "one frame per evs_step; consecutive steps overlapped on two streams (runtime.PipelinedSteps)"
    res["one_step_after_the_other"] = out["serial"]
    return res


# --------------------------------------------------------------------------- the reference's own CPU path
def _ref_worker(job):
    """One host process: the UNMODIFIED reference (baseline/_ref, evsim) stepping its
    cameras with generate_events_parallel(workers=1) + canonical_sort (the path
    SimNode runs every tick, orchestrator.py:160-172), plus the configured noise /
    accumulation.  Returns (frames done, seconds, events) of the timed part."""
    (cams, Wd, Hd, c, refr, cap, noise, accumulate, warm, frames, budget_s, start_at) = job
    sys.path.insert(0, REF_DIR)
    from evsim.bench.events_bench import _texture_frame
    from evsim.events import (EventCameraConfig, accumulate_events_to_image, canonical_sort, concat_batches,
                              generate_events_parallel, init_pixel_states, inject_noise_events)

    cfg = EventCameraConfig(c_pos=c, c_neg=c, refractory_us=refr, noise_rate_hz=noise, max_events_per_frame=cap)
    states = {s: init_pixel_states(_texture_frame(Wd, Hd, 0.137 * s, 0), cfg, seed=s) for s in cams}

    def one(s, k):
        fr = _texture_frame(Wd, Hd, 0.137 * s + k * DRIFT, k * TICK)
        b = generate_events_parallel(states[s], fr, (k - 1) * TICK, k * TICK, cfg, workers=1)
        if noise > 0:
            b = concat_batches([b, inject_noise_events(Wd, Hd, (k - 1) * TICK, k * TICK, noise, s * 1000 + k)])
        b = canonical_sort(b)
        if accumulate:
            accumulate_events_to_image(b, TICK, k * TICK, Wd, Hd)
        return len(b)

    k = 1
    for _ in range(warm):
        for s in cams:
            one(s, k)
        k += 1
    while time.time() < start_at:  # all processes start the timed part together
        time.sleep(0.001)
    n = nev = 0
    t0 = time.perf_counter()
    while n < frames * len(cams) and time.perf_counter() - t0 < budget_s:
        for s in cams:
            nev += one(s, k)
            n += 1
        k += 1
    return n, time.perf_counter() - t0, nev


def reference_throughput(cfg_key, warm, frames_per_proc, budget_s):
    """The reference's CPU path on all host cores: one process per core, cameras
    split over the processes (replica configs: one camera per process; sharded
    configs: the fixed stream set).  Returns (units/s, cores, sample text) or None
    when baseline/_ref is absent."""
    import multiprocessing as mpr

    if not os.path.isdir(os.path.join(REF_DIR, "evsim")):
        return None
    cfg = CONFIGS[cfg_key]
    cores = len(os.sched_getaffinity(0))
    if cfg["streams"]:
        nproc = min(cores, cfg["streams"])
        cams = [[s for s in range(cfg["streams"]) if s % nproc == i] for i in range(nproc)]
    else:
        nproc = cores
        cams = [[i] for i in range(nproc)]
    cap = cfg["cap_px"] * cfg["W"] * cfg["H"]
    # spawn + imports + warm-up frames (~1 s per HD frame on the reference path) before the common start
    start_at = time.time() + 8.0 + 1.5 * warm * (cfg["W"] * cfg["H"] / 1e6) * max(len(c) for c in cams)
    jobs = [(c, cfg["W"], cfg["H"], cfg["C"], cfg["refr"], cap, cfg["noise"], cfg_key in ("4", "5"), warm,
             frames_per_proc, budget_s, start_at) for c in cams]
    with mpr.get_context("spawn").Pool(nproc) as pool:
        res = pool.map(_ref_worker, jobs)
    n = sum(r[0] for r in res)
    secs = max(r[1] for r in res)
    nev = sum(r[2] for r in res)
    extra = {"4": " + inject_noise_events + accumulate_events_to_image",
             "5": " + accumulate_events_to_image"}.get(cfg_key, "")
    sample = (f"{n} {cfg['W']}x{cfg['H']} frames over {sum(len(c) for c in cams)} cameras on {nproc} processes "
              f"(one per host core), each through the unmodified reference (baseline/_ref evsim): "
              f"generate_events_parallel(workers=1){extra} + canonical_sort, {nev / secs / 1e6:.2f} Mev/s")
    return n / secs, nproc, sample


def port_throughput(seconds: float):
    """The oracle C port (banded pthreads, all host threads) on the HD workload:
    a second CPU figure next to the reference's own Python path."""
    import oracle

    oracle.build()
    cores = len(os.sched_getaffinity(0))
    st = oracle.init_state(oracle.texture_frame(W, H, 0.0), c_pos=C_TH, c_neg=C_TH, refractory_us=REFR, seed=0)
    frames = [oracle.texture_frame(W, H, k * DRIFT) for k in range(50)]
    oracle.generate(st, frames[1], 0, TICK, refractory_us=REFR, nthreads=cores)
    n = 0
    t0 = time.perf_counter()
    k = 2
    while time.perf_counter() - t0 < seconds:
        oracle.canonical_sort(oracle.generate(st, frames[k % 50], (k - 1) * TICK, k * TICK, refractory_us=REFR,
                                              nthreads=cores))
        n += 1
        k += 1
    return {"value": n / (time.perf_counter() - t0), "unit": "frames/s", "cores": cores, "kind": "port",
            "sample": f"{n} HD frames through oracle/evsim_oracle.c (banded pthreads) + canonical sort"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    T = args.frames_per_step or cfg["T"]
    sharded = cfg["streams"] is not None
    warm = min(args.warmup, 3)
    budget = 60.0
    r = reference_throughput(args.config, warm, args.steps, budget)
    if r is not None:
        value, cores, sample = r
        kind = "reference"
    else:  # the reference package is not installed: the oracle port stands in
        p = port_throughput(budget)
        value, cores, sample, kind = p["value"], p["cores"], p["sample"], "port"
    line = {
        "metric": cfg["metric"], "value": value, "unit": cfg["unit"], "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * T / value if value else None, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": config_dict(cfg, T, world, sharded),
        "cpu_baseline": {"value": value, "unit": cfg["unit"], "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": cfg["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg_key, seconds: float):
    """Reported CPU baseline for our line (rank 0, N=1): the reference's own path on
    all host cores on a bounded sample (~`seconds` of timed CPU work), else the port."""
    r = reference_throughput(cfg_key, 1, 10**6, seconds)
    if r is None:
        return port_throughput(seconds)
    value, cores, sample = r
    return {"value": value, "unit": CONFIGS[cfg_key]["unit"], "cores": cores, "kind": "reference", "sample": sample}


# --------------------------------------------------------------------------- our path
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2602_15018_b200 import _lib
    from paper_2602_15018_b200 import events as ev
    from paper_2602_15018_b200.distributed import shard_streams
    from paper_2602_15018_b200.runtime import StepEngine, StepShape
    from paper_2602_15018_b200.synth import PERIOD_FRAMES, texture_frame

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ck = args.config
    cfg = CONFIGS[ck]
    Wd, Hd, P = cfg["W"], cfg["H"], cfg["W"] * cfg["H"]
    T = args.frames_per_step or cfg["T"]
    K, Wm = args.steps, max(args.warmup, 3)
    cap = cfg["cap_px"] * P
    sharded = cfg["streams"] is not None
    streams = shard_streams(cfg["streams"], world, rank) if sharded else [rank]
    S = len(streams)
    ecfg = ev.EventCameraConfig(c_pos=cfg["C"], c_neg=cfg["C"], refractory_us=cfg["refr"],
                                noise_rate_hz=cfg["noise"])
    phases = [0.137 * s for s in streams]

    # frame windows [S][T][H][W] (contiguous), cycling a ring larger than L2
    if S == 1:
        ring_len = T * PERIOD_FRAMES // math.gcd(T, PERIOD_FRAMES)
        ring = device_texture_ring(Wd, Hd, ring_len, DRIFT, phases[0], dev)
        windows = [ring[j * T:(j + 1) * T][None] for j in range(ring_len // T)]
        ring_bytes = ring.numel() * 4
    else:
        ring = gpu_texture_windows(Wd, Hd, phases, T, dev)
        windows = [ring[j] for j in range(ring.shape[0])]
        ring_bytes = ring.numel() * 4
    states = [ev.init_pixel_states(ev.IntensityFrame(Wd, Hd, 0, texture_frame(Wd, Hd, ph)), ecfg, seed=s)
              for s, ph in zip(streams, phases)]
    uni = states[0].uniform_thresholds
    ref = torch.stack([s_.d_ref_log for s_ in states]).contiguous()
    last = torch.stack([s_.d_last_event_t for s_ in states]).contiguous()
    eng = StepEngine(StepShape(S, T, Hd, Wd, cap, _lib.EVS_ORDER_CANONICAL, TICK, ecfg.log_eps, cfg["refr"], uni),
                     dev)
    stream = torch.cuda.current_stream()
    state = {"k": 0}

    def step(stage_events=None):
        k = state["k"]
        eng.launch(windows[k % len(windows)], ref, last, t0=k * T * TICK, tick=TICK, validate=True, stream=stream,
                   stage_events=stage_events)
        state["k"] = k + 1

    for _ in range(Wm):
        step()
    torch.cuda.synchronize()
    counts, dropped, res, bad = eng.fetch_info()
    assert bad == _lib.NO_BAD and int(dropped.sum()) == 0

    # active pixels A_T and events E of one step for the bytes model (untimed)
    ref_before = ref.clone()
    step()
    torch.cuda.synchronize()
    A = int((ref != ref_before).sum().item())
    counts, _, _, _ = eng.fetch_info()
    E_step = int(counts.sum())

    # configs 4 and 5: the timed unit is more than the step (inside the timed region)
    extra = None
    if ck == "4":
        from paper_2602_15018_b200.simulator import EventSimulator, mix64

        sim = EventSimulator(Wd, Hd, streams=1, frames_per_step=T, config=ecfg, tick_us=TICK, device=dev)
        sim.reset([texture_frame(Wd, Hd, phases[0])], seeds=[streams[0]])

        def extra(k):  # one window: the step + its 5-bin voxel grid with the window's exact noise
            sim.step(windows[k % len(windows)])
            sim.voxel_window(0, bins=5, noise_seeds=[mix64(streams[0], 0x6E6F6973, k * T + f) for f in range(T)])
    elif ck == "5":
        from paper_2602_15018_b200.distributed import gather_keys, key32_layout, pack_segments

        lay = key32_layout(Wd, Hd, T * TICK)
        hist = torch.empty((S, Hd, Wd), dtype=torch.int64, device=dev)
        keybuf = torch.empty(S * T * cap, dtype=torch.int32, device=dev)
        L = _lib.load()
        gathered = {"n": 0}

        def extra(k):
            # the step, the signed histogram of every stream over the step window
            # (evs_step_histogram), then the step's events as packed 4-byte keys
            # (evs_pack_segments) gathered to rank 0 over NCCL
            import ctypes

            step()
            t_end = (k + 1) * T * TICK
            rc = L.evs_step_histogram(ctypes.byref(eng.params), ctypes.byref(eng.bufs), eng.workspace.data_ptr(),
                                      eng.workspace.numel(), T * TICK, t_end, hist.data_ptr(), _lib.stream_ptr())
            _lib.check(rc, "evs_step_histogram")
            keys, offs = pack_segments(eng.info[0], (eng.ev_t, eng.ev_x, eng.ev_y, eng.ev_p), k * T * TICK, lay, 4,
                                       out=keybuf)
            n = int(offs[-1].item())
            if world > 1:
                out, _ = gather_keys(keys[:n], dst=0)
                gathered["n"] = out.numel() if out is not None else 0
            else:
                gathered["n"] = n

    # timed region
    runner = eng
    if extra is None:
        # CUDA graph of G steps (one per window); the step clock advances on the device
        G = max(g for g in range(1, min(K, 64) + 1) if K % g == 0 and (g % len(windows) == 0 or g < len(windows)))
        k_next = state["k"]
        if args.pipelined and G % 2 == 0:
            from paper_2602_15018_b200.runtime import PipelinedSteps

            runner = PipelinedSteps(eng.shape, dev)
            runner.engines[0] = eng
            for _ in range(2):  # (kernel attributes of the second engine) -- untimed
                runner.engines[1].launch(windows[state["k"] % len(windows)], ref, last, t0=state["k"] * T * TICK,
                                         tick=TICK, validate=True, stream=stream)
                state["k"] += 1
            k_next = state["k"]
        runner.capture([windows[(k_next + i) % len(windows)] for i in range(G)], ref, last, tick=TICK,
                       t0=k_next * T * TICK)
        reps = K // G
        launches = K * 5 + reps
    else:
        reps = K
        launches = None
        for w in range(2):  # warm the extras
            extra(state["k"] if ck == "5" else w)
        if ck == "4":
            sim.result()  # (untimed) a fetched step: the next steps' tile groups follow its density
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if extra is None:
        for _ in range(reps):
            runner.replay()
        state["k"] += K
    else:
        for i in range(K):
            extra(state["k"] if ck == "5" else 2 + i)
    e1.record(stream)
    torch.cuda.synchronize()
    sampler.stop()
    ms = e0.elapsed_time(e1)
    counts, dropped, _, bad = eng.fetch_info()
    assert bad == _lib.NO_BAD and int(dropped.sum()) == 0
    E_last = int(counts.sum())
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tot = torch.tensor([S * T, E_last, A, E_step], dtype=torch.float64, device=dev)
        dist.all_reduce(tot)
        units_step, E_all, A_all, E_step_all = [float(v) for v in tot.tolist()]
        dist.barrier()
    else:
        units_step, E_all, A_all, E_step_all = S * T, E_last, A, E_step

    # per-stage device time (profiled pass, same steps, outside the headline region)
    nprof = min(K, 100)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(nprof)]
    for row in evs:
        for e in row:
            e.record(stream)
    torch.cuda.synchronize()
    for row in evs:
        step(stage_events=row)
    torch.cuda.synchronize()
    stage = np.array([[row[i].elapsed_time(row[i + 1]) for i in range(4)] for row in evs])
    stage_ms = stage.mean(axis=0)

    value = units_step * K / (ms / 1e3)
    ev_s = E_all * K / (ms / 1e3)
    peak, peak_kind = measured_peak_hbm()
    B = algorithmic_bytes(P, A_all, E_step_all, cfg["refr"], uni is not None, T, S=int(units_step // T))
    step_ms = ms / K
    achieved = B / (step_ms / 1e3) / 1e9
    gen_bytes = (4 * P * T + 4 * P) * int(units_step // T) + 20 * A_all + 8 * E_step_all  # K1's own traffic model
    gen_achieved = gen_bytes / (stage_ms[1] / 1e3) / 1e9 / (world if world > 1 else 1)
    traffic = None
    try:  # ncu dram bytes of one step of this workload (committed profile)
        with open(os.path.join(ROOT, "profiles", "step_traffic.json")) as fh:
            tr = json.load(fh)
        if ck == "2" and int(tr["frames_per_step"]) == T:
            traffic = int(tr["bytes_per_step"])
    except Exception:
        traffic = None

    e2e = e2e_frame = per_frame = self_check = None
    if ck == "2":
        # end to end through the public APIs with HOST buffers, copies inside the timed
        # region: EventSimulator.run_host (T frames in, T host batches out, pipelined)
        from paper_2602_15018_b200.simulator import EventSimulator

        host_frames = np.stack([texture_frame(W, H, phases[0] + k * DRIFT) for k in range(PERIOD_FRAMES)])
        sim = EventSimulator(W, H, streams=1, frames_per_step=T, config=ecfg, tick_us=TICK, device=dev)
        sim.reset([host_frames[0]], seeds=[rank])
        win_host = [np.ascontiguousarray(host_frames[np.arange(j * T, j * T + T) % PERIOD_FRAMES][None])
                    for j in range(max(1, PERIOD_FRAMES // math.gcd(T, PERIOD_FRAMES)))]
        for w in win_host:  # page-locked source windows (a renderer would write into these)
            EventSimulator.pin_host(w)
        for _ in sim.run_host([win_host[j % len(win_host)] for j in range(4)]):
            pass
        torch.cuda.synchronize()
        ke_steps = max(4, min(K, 40))
        d2h = 0
        t0 = time.perf_counter()
        for out in sim.run_host(win_host[j % len(win_host)] for j in range(ke_steps)):
            d2h += sum(13 * len(b) for b in out[0])
            del out
        e2e_s = time.perf_counter() - t0
        for w in win_host:
            EventSimulator.unpin_host(w)
        e2e_v = torch.tensor([ke_steps * T / e2e_s], dtype=torch.float64, device=dev)
        if world > 1:  # slowest rank sets the pace: world x its rate
            dist.all_reduce(e2e_v, op=dist.ReduceOp.MIN)
        e2e = {"value": world * float(e2e_v.item()), "unit": "frames/s", "h2d_bytes_per_step": 4 * P * T,
               "d2h_bytes_per_step": int(d2h / ke_steps),
               "api": f"paper_2602_15018_b200.simulator.EventSimulator.run_host (page-locked host numpy "
                      f"[1,{T},H,W] windows in, host EventBatch per frame out; H2D/D2H overlapped with compute)",
               "frames_per_step": T}
        st2 = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, host_frames[0]), ecfg, seed=rank)
        ke = max(10, min(K, 200))
        for k in range(1, 4):
            ev.generate_events_parallel(st2, ev.IntensityFrame(W, H, k * TICK, host_frames[k % 50]),
                                        (k - 1) * TICK, k * TICK, ecfg)
        torch.cuda.synchronize()
        d2h = 0
        t0 = time.perf_counter()
        for k in range(4, 4 + ke):
            b = ev.generate_events_parallel(st2, ev.IntensityFrame(W, H, k * TICK, host_frames[k % 50]),
                                            (k - 1) * TICK, k * TICK, ecfg)
            d2h += 13 * len(b)
        torch.cuda.synchronize()
        e2e_frame = {"value": world * ke / (time.perf_counter() - t0), "unit": "frames/s",
                     "h2d_bytes_per_step": 4 * P, "d2h_bytes_per_step": int(d2h / ke),
                     "api": "paper_2602_15018_b200.events.generate_events_parallel (drop-in, one frame per call)"}
        # self-check of the timed launch shape against the oracle fixture (untimed)
        mism = verify_launch_shape(dev, T, pipelined=bool(args.pipelined))
        self_check = {"fixture": "tests/golden/bench_hd_t50.json (oracle, 150 HD frames: per-frame counts, drops, "
                                 "reservations, SHA-1 of the canonical events; final state)",
                      "launch": f"same StepShape (T={T}), eager step then CUDA-graph replays"
                                + (" of two engines on two streams (PipelinedSteps)" if args.pipelined else ""),
                      "frames": 150,
                      "mismatches": [str(m) for m in mism[:10]], "ok": not mism}
        if T != 1 and args.compare_t1:
            per_frame = measure_t1(args, dev, ecfg, phases[0], rank)
            per_frame["pixel_major_order"] = measure_t1(args, dev, ecfg, phases[0], rank,
                                                        _lib.EVS_ORDER_PIXEL_MAJOR)
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    cpu = cpu_baseline(ck, args.cpu_seconds) if world == 1 and args.cpu_seconds > 0 else None
    clocks = sampler.summary()
    line = {
        "metric": cfg["metric"], "value": value, "unit": cfg["unit"], "n_gpus": world, "steps": K,
        "warmup": Wm, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, T, world, sharded),
        "mevents_per_s": ev_s / 1e6, "events_per_frame": E_step_all / units_step, "active_px_per_step": A_all,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak / (world if world > 1 else 1), "traffic": traffic,
                     "peak_kind": peak_kind,
                     "traffic_note": "ncu dram read+write bytes per step (profiles/step_traffic.json), config 2 only",
                     "kernel": "evs_step (k_prologue + k_generate + k_group_hist + k_tilescan + k_tile_order), "
                               "device time per step of the timed region (per GPU)",
                     "algorithmic_bytes_per_step": B,
                     "stage_ms_per_step": {"prologue": stage_ms[0], "generate": stage_ms[1],
                                           "group_hist+tilescan": stage_ms[2], "order": stage_ms[3]},
                     "generate_only": {"bytes": gen_bytes, "achieved": gen_achieved,
                                       "frac": gen_achieved / peak}},
        "ring_bytes": ring_bytes,
        "cpu_baseline": cpu,
        "gpu_launches": launches if launches is not None else f"{K} steps x (5 step kernels + extras)",
        "clocks": clocks,
    }
    if ck == "2":
        line.update({"per_frame_launch": per_frame, "e2e": e2e, "e2e_per_frame_api": e2e_frame,
                     "self_check": self_check})
    if ck == "5":
        line["gather"] = {"keys_on_rank0_last_step": gathered["n"], "key_bytes": 4, "layout_bits": lay}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if self_check is not None and not self_check["ok"]:
        print(f"bench self-check FAILED: frames {self_check['mismatches']} differ from the oracle fixture",
              file=sys.stderr)
        sys.exit(1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--frames-per-step", type=int, default=0, help="0: the config's default (HD: 50)")
    ap.add_argument("--config", default="2", choices=sorted(CONFIGS))
    ap.add_argument("--compare-t1", type=int, default=1)
    ap.add_argument("--pipelined", type=int, default=1,
                    help="1: consecutive steps on two engines / streams (runtime.PipelinedSteps)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
