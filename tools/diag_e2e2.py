"""Diagnostic: run_host pipeline timing (HD, T=50) and raw PCIe rates."""
import sys, os, time, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_15018_b200 import events as ev
from paper_2602_15018_b200.simulator import EventSimulator
from paper_2602_15018_b200.synth import texture_frame
W, H, T = 1280, 720, 50
dev = torch.device("cuda")
cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
host = np.stack([texture_frame(W, H, 0.02 * k) for k in range(50)])
win = [np.ascontiguousarray(host[None])]
for w in win: EventSimulator.pin_host(w)
sim = EventSimulator(W, H, 1, T, cfg)
sim.reset([host[0]], seeds=[0])
for _ in sim.run_host([win[0]] * 2): pass
torch.cuda.synchronize()
n = 10
t0 = time.perf_counter()
for out in sim.run_host(win[0] for _ in range(n)):
    del out
dt = time.perf_counter() - t0
print(f"run_host: {dt / n * 1e3:.2f} ms per window, {n * T / dt:.0f} frames/s")
# raw rates
d = torch.empty(host.nbytes // 4, dtype=torch.float32, device=dev)
src = torch.from_numpy(win[0].reshape(-1))
for _ in range(2): d.copy_(src, non_blocking=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): d.copy_(src, non_blocking=True)
torch.cuda.synchronize(); r = (time.perf_counter() - t0) / 5
print(f"H2D pinned {win[0].nbytes/1e6:.0f} MB: {r*1e3:.2f} ms = {win[0].nbytes/r/1e9:.1f} GB/s")
hb = torch.empty(420_000_000, dtype=torch.uint8, pin_memory=True)
db = torch.empty(420_000_000, dtype=torch.uint8, device=dev)
for _ in range(2): hb.copy_(db, non_blocking=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): hb.copy_(db, non_blocking=True)
torch.cuda.synchronize(); r = (time.perf_counter() - t0) / 5
print(f"D2H pinned 420 MB: {r*1e3:.2f} ms = {0.42/r:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): hb.copy_(db, non_blocking=True)
    with torch.cuda.stream(s2): d.copy_(src, non_blocking=True)
torch.cuda.synchronize(); r = (time.perf_counter() - t0) / 5
print(f"H2D || D2H: {r*1e3:.2f} ms")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for out in sim.run_host(win[0] for _ in range(5)):
    del out
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
