"""Diagnostic (RES=WxH, ORDER=pixel|canonical pseudo-variables): per-stage device times of one-frame steps (T=1), HD bench workload.

  python tools/diag_t1.py [variant ...]    variant = ENV=VAL[,ENV=VAL] (e.g. EVS_GT=4)
Per variant: stage times (events between stages) and back-to-back frame time.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2602_15018_b200 import _lib, events as ev
from paper_2602_15018_b200.runtime import StepEngine, StepShape
from paper_2602_15018_b200.synth import texture_frame

dev = torch.device("cuda", 0)
cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)


def run(variant):
    env = dict(kv.split("=", 1) for kv in variant.split(",") if kv)
    W, H = map(int, env.pop("RES", "1280x720").split("x"))
    order = _lib.EVS_ORDER_PIXEL_MAJOR if env.pop("ORDER", "canonical") == "pixel" else _lib.EVS_ORDER_CANONICAL
    ring = bench.device_texture_ring(W, H, 50, 0.02, 0.0, dev)
    for k, v in env.items():
        os.environ[k] = v
    st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, 0.0)), cfg, seed=0)
    eng = StepEngine(StepShape(1, 1, H, W, 8 * W * H, order, 1000, 0.01, 100,
                               st.uniform_thresholds), dev)
    rows = []
    k = 0
    for _ in range(60):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        for e in evs:
            e.record()  # (torch's bookkeeping; the library re-records them between stages)
        eng.launch(ring[k % 50:k % 50 + 1], st.d_ref_log, st.d_last_event_t, t0=k * 1000, tick=1000,
                   stage_events=evs)
        k += 1
        torch.cuda.synchronize()
        rows.append([evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(4)])
    r = np.array(rows[10:])
    eng.capture([ring[(k + i) % 50:(k + i) % 50 + 1] for i in range(50)], st.d_ref_log, st.d_last_event_t,
                tick=1000, t0=k * 1000)
    eng.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 4
    e0.record()
    for _ in range(n):
        eng.replay()
    e1.record()
    torch.cuda.synchronize()
    n *= 50
    per = e0.elapsed_time(e1) * 1e3 / n
    print(f"{variant or 'default':24s} stage us (prologue, generate, tilescan, order) median",
          np.round(np.median(r, 0), 1), f" graph {per:.1f} us/frame", flush=True)
    for k in env:
        os.environ.pop(k)


for v in (sys.argv[1:] or [""]):
    run(v)
