"""Diagnostic: per-window wall times of EventSimulator.run_host (HD, T=50, bench windows)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_15018_b200 import events as ev
from paper_2602_15018_b200.simulator import EventSimulator
from paper_2602_15018_b200.synth import texture_frame

W, H, T = 1280, 720, 50
cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
host = np.stack([texture_frame(W, H, 0.02 * k) for k in range(50)])
win = np.ascontiguousarray(host[None])
EventSimulator.pin_host(win)
sim = EventSimulator(W, H, 1, T, cfg)
sim.reset([host[0]], seeds=[0])
for rep in range(3):
    for _ in sim.run_host([win] * 4):
        pass
    torch.cuda.synchronize()
    ts = [time.perf_counter()]
    for out in sim.run_host(win for _ in range(40)):
        del out
        ts.append(time.perf_counter())
    d = np.diff(ts) * 1e3
    print(f"rep {rep}: total {ts[-1] - ts[0]:.3f} s = {40 * T / (ts[-1] - ts[0]):.0f} fps; window ms "
          f"median {np.median(d):.2f} min {d.min():.2f} max {d.max():.2f}; first {d[0]:.2f}; "
          f"slow(>1.5x median) {int((d > 1.5 * np.median(d)).sum())}", flush=True)
    print("   ", np.round(d, 1).tolist(), flush=True)
