#!/usr/bin/env python
"""Measure the other BASELINE.json configs on one B200 (bench.py covers config 2).

  config 1: DAVIS 346x260, C=0.2, 1000 moving-texture frames (+ the CPU reference port)
  config 3: 64 independent 640x480 cameras, C=0.2 (camera-frames/s, one GPU's share)
  config 4: 1920x1080, C=0.05 (multi-crossing), 10 Hz noise merged per frame, 5-bin
            voxel grid per 20-frame window
  config 5: 256 DAVIS streams (32 per GPU at N=8; here all 256 on one GPU), signed
            histogram of every stream's last frame

Device time with CUDA events around the timed steps (inputs resident in HBM,
frame ring > L2 where it matters); algorithmic bytes per SURVEY.md 8(d).
Writes one JSON object per config to stdout.

  python tools/bench_configs.py [--configs 1,3,4,5] [--cpu-seconds 10]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TICK = 1000
DRIFT = 0.02


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def ring(W, H, n, phases, dev):
    """[S, n, H, W] texture frames on the GPU (f64 math, f32 out, events_bench.py:19-26)."""
    import torch

    x = torch.arange(W, dtype=torch.float64, device=dev) / W
    y = torch.arange(H, dtype=torch.float64, device=dev) / H
    grid = y[:, None] * 2.0 + x[None, :] * 3.0
    out = torch.empty((len(phases), n, H, W), dtype=torch.float32, device=dev)
    for s, ph in enumerate(phases):
        for k in range(n):
            out[s, k] = (0.5 + 0.45 * torch.sin(2.0 * math.pi * (grid + (ph + k * DRIFT)))).to(torch.float32)
    return out


def run_batched(W, H, S, T, c, refr, steps, warm, dev, noise_hz=0.0):
    """EventSimulator steps over a device frame ring; returns timing + event stats."""
    import torch

    from paper_2602_15018_b200 import events as ev
    from paper_2602_15018_b200.simulator import EventSimulator
    from paper_2602_15018_b200.synth import texture_frame

    phases = [0.137 * s for s in range(S)]
    nring = max(T, 50 // math.gcd(T, 50) * T if T < 50 else T)
    fr = ring(W, H, nring, phases, dev)
    nwin = nring // T
    cfg = ev.EventCameraConfig(c_pos=c, c_neg=c, refractory_us=refr, noise_rate_hz=noise_hz)
    sim = EventSimulator(W, H, streams=S, frames_per_step=T, config=cfg, device=dev)
    sim.reset([texture_frame(W, H, ph) for ph in phases], seeds=list(range(S)))
    P = W * H
    ref0 = sim.ref.clone()
    for i in range(warm):
        sim.step(fr[:, (i % nwin) * T:(i % nwin + 1) * T])
    torch.cuda.synchronize()
    A = int((sim.ref != ref0).sum().item())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        sim.step(fr[:, ((warm + i) % nwin) * T:((warm + i) % nwin + 1) * T])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    res = sim.result()
    E = float(res.counts.sum())  # events of the last step (all segments)
    B = 4 * P * T * S + 4 * P * S + 12 * min(A, S * P) + (8 * min(A, S * P) if refr else 0) + 13 * E
    return {"ms_per_step": ms, "frames_per_step": S * T, "events_per_step": E, "bytes_per_step": B,
            "frames_per_s": S * T / (ms / 1e3), "mevents_per_s": E / (ms / 1e3) / 1e6,
            "achieved_gbs": B / (ms / 1e3) / 1e9}, sim


def cpu_port(W, H, c, refr, frames, seconds, phases=(0.0,)):
    """The oracle C port (all host threads) on a bounded sample."""
    import oracle

    oracle.build()
    cores = len(os.sched_getaffinity(0))
    n = 0
    nev = 0
    t0 = time.perf_counter()
    for ph in phases:
        st = oracle.init_state(oracle.texture_frame(W, H, ph), c_pos=c, c_neg=c, refractory_us=refr, seed=0)
        for k in range(1, frames + 1):
            b = oracle.canonical_sort(oracle.generate(st, oracle.texture_frame(W, H, ph + k * DRIFT),
                                                      (k - 1) * TICK, k * TICK, refractory_us=refr,
                                                      nthreads=cores))
            n += 1
            nev += len(b)
            if time.perf_counter() - t0 > seconds:
                break
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    return {"frames_per_s": n / dt, "mevents_per_s": nev / dt / 1e6, "cores": cores, "frames": n,
            "kind": "port (oracle/evsim_oracle.c, banded pthreads)"}


def main():
    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    pk = peak()
    want = set(args.configs.split(","))
    out = []
    if "1" in want:
        W, H = 346, 260
        r, _ = run_batched(W, H, 1, 50, 0.2, 0, steps=20, warm=3, dev=dev)
        line = {"config": 1, "workload": "DAVIS 346x260, C=0.2, 1000 frames (20 steps x 50 frames), 1 stream",
                **r, "roofline_frac": r["achieved_gbs"] / pk}
        if args.cpu_seconds > 0:
            line["cpu_baseline"] = cpu_port(W, H, 0.2, 0, 1000, args.cpu_seconds)
        out.append(line)
    if "3" in want:
        W, H = 640, 480
        r, _ = run_batched(W, H, 64, 4, 0.2, 0, steps=10, warm=3, dev=dev)
        line = {"config": 3, "workload": "64 x 640x480 cameras, C=0.2, 4 frames per step (one GPU)",
                **r, "camera_frames_per_s": r["frames_per_s"], "roofline_frac": r["achieved_gbs"] / pk}
        if args.cpu_seconds > 0:
            line["cpu_baseline"] = cpu_port(W, H, 0.2, 0, 5, args.cpu_seconds,
                                            phases=[0.137 * s for s in range(64)])
        out.append(line)
    if "4" in want:
        from paper_2602_15018_b200 import events as ev
        from paper_2602_15018_b200.noise import noise_params, run_noise
        from paper_2602_15018_b200.represent import canonical_sort, merge_canonical, voxel_grid
        from paper_2602_15018_b200.events.types import DeviceEventBatch
        from paper_2602_15018_b200.simulator import mix64

        W, H, T = 1920, 1080, 20
        r, sim = run_batched(W, H, 1, T, 0.05, 0, steps=5, warm=2, dev=dev, noise_hz=10.0)
        # full per-window pipeline: step + per-frame exact noise + 5-bin voxel of the window
        fr = ring(W, H, T, [0.5], dev)
        nwin = 5
        sim.step(fr[:, :T])
        sim.voxel_window(0, bins=5, noise_seeds=[mix64(7, 0x6E6F6973, f) for f in range(T)])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for w in range(nwin):
            sim.step(fr[:, :T])
            vox = sim.voxel_window(0, bins=5, noise_seeds=[mix64(7, 0x6E6F6973, (w + 1) * T + f) for f in range(T)])
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / nwin
        # the same window with canonical signal+noise event batches per frame (merge-path), then the voxel
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nwin2 = 2
        for w in range(nwin2):
            sim.step(fr[:, :T])
            t_end = sim.t_next
            grids = []
            for f in range(T):
                sig = sim.segment(0, f)
                t_now = t_end - (T - 1 - f) * TICK
                p = noise_params(W, H, t_now - TICK, t_now, 10.0, mix64(7, 0x6E6F6973, w * T + f), order=0)
                n, b = run_noise(p, dev)
                nz = canonical_sort(DeviceEventBatch(b["t"][:n], b["x"][:n], b["y"][:n], b["p"][:n], 0, False))
                merged = merge_canonical(sig, nz)
                grids.append(voxel_grid(merged, t_end - T * TICK, t_end, W, H, bins=5, device_output=True))
            torch.stack(grids).sum(0)
        torch.cuda.synchronize()
        wall2 = (time.perf_counter() - t0) / nwin2
        out.append({"config": 4, "workload": "1920x1080, C=0.05, 20-frame windows", **r,
                    "roofline_frac": r["achieved_gbs"] / pk,
                    "with_noise_and_voxel": {"ms_per_window_wall": wall * 1e3, "frames_per_s": T / wall,
                                             "note": "EventSimulator.voxel_window: step + exact 10 Hz noise per "
                                                     "frame + one 5-bin voxel grid per 20-frame window "
                                                     "(signal voxel from the tile regions, noise added by a segmented accumulation, one host read per window)",
                                             "voxel_sum": float(vox.sum().item())},
                    "with_merged_event_batches": {"ms_per_window_wall": wall2 * 1e3, "frames_per_s": T / wall2,
                                                  "note": "per frame: noise, canonical sort, merge-path into the "
                                                          "signal segment, voxel (host-driven, synchronising)"}})
    if "5" in want:
        W, H = 346, 260
        r, sim = run_batched(W, H, 256, 4, 0.2, 0, steps=10, warm=3, dev=dev)
        sim.histograms(20 * TICK)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            hist = sim.histograms(4 * TICK)  # every stream's last 4-frame window
        e1.record()
        torch.cuda.synchronize()
        hist_ms = e0.elapsed_time(e1) / 10
        out.append({"config": 5, "workload": "256 x DAVIS 346x260 streams, C=0.2, 4 frames per step (one GPU)",
                    **r, "camera_frames_per_s": r["frames_per_s"], "roofline_frac": r["achieved_gbs"] / pk,
                    "histograms_256_streams_ms": hist_ms,
                    "histogram_note": "EventSimulator.histograms: accumulate_events_to_image of all 256 streams' "
                                      "step windows in one launch (device time)",
                    "hist_abs_sum": int(hist.abs().sum().item())})
    for line in out:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
