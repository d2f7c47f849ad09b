"""Diagnostic: config-4 window costs (1080p, C=0.05, T=20): step, voxel of the
signal, voxel with per-frame noise; device time with CUDA events + wall."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench_configs import ring  # noqa: E402
from paper_2602_15018_b200 import events as ev
from paper_2602_15018_b200.simulator import EventSimulator, mix64
from paper_2602_15018_b200.synth import texture_frame

W, H, T = 1920, 1080, 20
dev = torch.device("cuda", 0)
cfg = ev.EventCameraConfig(c_pos=0.05, c_neg=0.05, refractory_us=0, noise_rate_hz=10.0)
sim = EventSimulator(W, H, streams=1, frames_per_step=T, config=cfg, device=dev)
sim.reset([texture_frame(W, H, 0.5)], seeds=[0])
fr = ring(W, H, T, [0.5], dev)


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, (time.perf_counter() - w0) * 1e3 / n


k = [0]


def seeds():
    k[0] += 1
    return [mix64(7, 0x6E6F6973, k[0] * T + f) for f in range(T)]


print("step            ms (device, wall)", timed(lambda: sim.step(fr[:, :T])))
print("voxel signal    ms", timed(lambda: sim.voxel_window(0, bins=5)))
print("voxel +noise    ms", timed(lambda: sim.voxel_window(0, bins=5, noise_seeds=seeds())))
print("step+vox+noise  ms", timed(lambda: (sim.step(fr[:, :T]), sim.voxel_window(0, bins=5, noise_seeds=seeds()))))
print("histograms ms", timed(lambda: sim.histograms(20 * 1000)))
