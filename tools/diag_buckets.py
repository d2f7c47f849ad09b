"""Diagnostic: events per 8-us t_rel bucket in the bench's steady state, and K2 time."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2602_15018_b200 import _lib, events as ev
from paper_2602_15018_b200.runtime import StepEngine, StepShape
from paper_2602_15018_b200.synth import texture_frame
W, H, T = 1280, 720, 25
dev = torch.device("cuda", 0)
ring = bench.device_texture_ring(W, H, 50, 0.02, 0.0, dev)
cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, 0.0)), cfg, seed=0)
eng = StepEngine(StepShape(1, T, H, W, 8 * W * H, _lib.EVS_ORDER_CANONICAL, 1000, 0.01, 100, st.uniform_thresholds), dev)
for k in range(30):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    [e.record() for e in evs]
    eng.launch(ring[(k % 2) * T:(k % 2 + 1) * T], st.d_ref_log, st.d_last_event_t, t0=k * T * 1000, tick=1000, stage_events=evs)
    torch.cuda.synchronize()
    if k in (0, 1, 5, 29):
        print(k, "stage ms", [round(evs[i].elapsed_time(evs[i + 1]), 3) for i in range(4)])
counts, dropped, res, bad = eng.fetch_info()
for seg in (0, 12, 24):
    n = int(counts[seg])
    t = eng.ev_t[seg, :n].cpu().numpy()
    tr = t - t.min()
    hb = np.bincount(tr // 8)
    print("seg", seg, "events", n, "buckets>0", (hb > 0).sum(), "max bucket", hb.max(), "n>12288", (hb > 12288).sum())
