"""Per-call time split of the drop-in generate_events_parallel (HD, host numpy in / out)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_15018_b200 import events as ev
from paper_2602_15018_b200.events import model as M
from paper_2602_15018_b200.runtime import d2h_rows, upload_frame
from paper_2602_15018_b200.synth import texture_frame

W, H = 1280, 720
cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
frames = [texture_frame(W, H, 0.02 * k) for k in range(60)]
st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, frames[0]), cfg, seed=0)
for k in range(1, 10):
    ev.generate_events_parallel(st, ev.IntensityFrame(W, H, k * 1000, frames[k]), (k - 1) * 1000, k * 1000, cfg)
torch.cuda.synchronize()
n = 40
t0 = time.perf_counter()
for k in range(10, 10 + n):
    b = ev.generate_events_parallel(st, ev.IntensityFrame(W, H, k * 1000, frames[k % 60]), (k - 1) * 1000, k * 1000, cfg)
t1 = time.perf_counter()
print(f"generate_events_parallel: {(t1 - t0) / n * 1e6:.0f} us/frame ({n / (t1 - t0):.0f} frames/s), {len(b)} events")
# pieces
dev = st.device
tu = time.perf_counter()
for k in range(n):
    d = upload_frame(frames[k % 60], dev, st._ctx)
torch.cuda.synchronize()
print(f"upload_frame: {(time.perf_counter() - tu) / n * 1e6:.0f} us")
eng = M._engine(st, cfg, 1, 1000)
tl = time.perf_counter()
for k in range(n):
    eng.launch(d, st.d_ref_log, st.d_last_event_t, st.d_thresholds_pos, st.d_thresholds_neg, t_bounds=None,
               t0=(100 + k) * 1000, tick=1000, validate=True)
    c, dr, r, bad = eng.fetch_info()
print(f"launch + fetch_info: {(time.perf_counter() - tl) / n * 1e6:.0f} us")
from paper_2602_15018_b200.runtime import PinnedPool
pool = PinnedPool()
m = int(c[0])
td = time.perf_counter()
for k in range(n):
    t, x, y, p = d2h_rows(pool, m, [eng.ev_t[0], eng.ev_x[0], eng.ev_y[0], eng.ev_p[0]])
print(f"d2h_rows ({m} events): {(time.perf_counter() - td) / n * 1e6:.0f} us")
