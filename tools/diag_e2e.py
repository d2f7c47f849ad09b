"""Diagnostic: where the per-frame drop-in API time goes (HD, C=0.15, refr 100)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_15018_b200 import events as ev
from paper_2602_15018_b200.synth import texture_frame
W, H = 1280, 720
cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
frames = [texture_frame(W, H, 0.02 * k) for k in range(50)]
st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, frames[0]), cfg, seed=0)
for k in range(1, 5):
    ev.generate_events_parallel(st, ev.IntensityFrame(W, H, k * 1000, frames[k % 50]), (k - 1) * 1000, k * 1000, cfg)
torch.cuda.synchronize()
N = 100
t0 = time.perf_counter()
for k in range(5, 5 + N):
    b = ev.generate_events_parallel(st, ev.IntensityFrame(W, H, k * 1000, frames[k % 50]), (k - 1) * 1000, k * 1000, cfg)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / N
print(f"api per frame {dt*1e3:.3f} ms  ({1/dt:.0f} FPS), events {len(b)}")
# pieces
dev = torch.device("cuda")
x = torch.empty(len(b), dtype=torch.int64, device=dev)
y16 = torch.empty(len(b), dtype=torch.int16, device=dev)
torch.cuda.synchronize()
for name, fn in [
    ("h2d 3.7MB pageable", lambda: torch.from_numpy(frames[1]).to(dev)),
    ("numpy->pinned->dev", None),
    ("d2h t int64 pageable", lambda: x.cpu()),
    ("d2h x int16 pageable", lambda: y16.cpu()),
]:
    if fn is None:
        pin = torch.empty((H, W), dtype=torch.float32, pin_memory=True)
        def fn():
            pin.numpy()[...] = frames[1]
            return pin.to(dev, non_blocking=True)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20): fn()
    torch.cuda.synchronize()
    print(f"{name:24s} {(time.perf_counter()-t0)/20*1e3:.3f} ms")
pin_t = torch.empty(len(b), dtype=torch.int64, pin_memory=True)
for _ in range(3): pin_t.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    pin_t.copy_(x, non_blocking=True); torch.cuda.synchronize(); a = pin_t.numpy().copy()
print(f"{'d2h t pinned+copy':24s} {(time.perf_counter()-t0)/20*1e3:.3f} ms")
t0 = time.perf_counter()
for _ in range(20):
    a = np.add(np.arange(len(b), dtype=np.uint16), np.uint64(12345), dtype=np.uint64)
print(f"{'host t rebuild':24s} {(time.perf_counter()-t0)/20*1e3:.3f} ms")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for k in range(200, 220):
    b = ev.generate_events_parallel(st, ev.IntensityFrame(W, H, k * 1000, frames[k % 50]), (k - 1) * 1000, k * 1000, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
