"""K1 time on a static scene (no pixel active: per-frame fixed costs only) vs
the moving texture (fixed + per-active-pixel work), HD, T=50."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2602_15018_b200 import _lib, events as ev
from paper_2602_15018_b200.runtime import StepEngine, StepShape
from paper_2602_15018_b200.synth import texture_frame

W, H, T = 1280, 720, 50
dev = torch.device("cuda")
cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
for name in ("static", "texture"):
    st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, 0.0)), cfg, seed=0)
    ring = bench.device_texture_ring(W, H, T, 0.02, 0.0, dev)
    if name == "static":
        ring[:] = ring[0]
    eng = StepEngine(StepShape(1, T, H, W, 8 * W * H, 1, 1000, 0.01, 100, st.uniform_thresholds), dev)
    times = []
    for k in range(12):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        for e in evs:
            e.record()
        eng.launch(ring, st.d_ref_log, st.d_last_event_t, t0=k * T * 1000, tick=1000, stage_events=evs)
        torch.cuda.synchronize()
        if k >= 2:
            times.append([evs[i].elapsed_time(evs[i + 1]) for i in range(4)])
    import numpy as np
    t = np.mean(times, axis=0)
    c, _, _, _ = eng.fetch_info()
    print(name, "events/frame", int(c.sum()) / T, "stage ms", [round(x, 4) for x in t])
