"""Diagnostic: per-step stage times over a long run (bench workload), incl. after graph replays."""
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
times = []
nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 120
for k in range(nsteps):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    [e.record() for e in evs]
    eng.launch(ring[(k % 2) * T:(k % 2 + 1) * T], st.d_ref_log, st.d_last_event_t, t0=k * T * 1000, tick=1000, stage_events=evs)
    torch.cuda.synchronize()
    times.append([evs[i].elapsed_time(evs[i + 1]) for i in range(4)])
    if k % 10 == 0 or k > nsteps - 4:
        counts, dropped, res, bad = eng.fetch_info()
        mx = 0
        for seg in range(T):
            n = int(counts[seg])
            if n == 0: continue
            t = eng.ev_t[seg, :n].cpu().numpy()
            hb = np.bincount((t - t.min()) // 8); mx = max(mx, hb.max())
        print(k, "stage ms", [round(x, 3) for x in times[-1]], "events", int(counts.sum()), "max bucket", mx, flush=True)
