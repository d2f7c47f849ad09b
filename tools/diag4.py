"""Diagnostic: slow-pixel counts per segment (EVS_FAST_DBG=3 puts them in the reservation counts)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["EVS_FAST_DBG"] = "3"
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
for k in range(4):
    eng.launch(ring[(k % 2) * T:(k % 2 + 1) * T], st.d_ref_log, st.d_last_event_t, t0=k * T * 1000, tick=1000)
    torch.cuda.synchronize()
    counts, dropped, res, bad = eng.fetch_info()
    print(k, "events/seg", int(counts.mean()), "slow+res per seg", res[:6], "mean", res.mean())
