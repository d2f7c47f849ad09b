import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2602_15018_b200 import _lib, events as ev
from paper_2602_15018_b200.runtime import StepEngine, StepShape, PinnedPool, d2h_compact, d2h_segments
from paper_2602_15018_b200.synth import texture_frame
W, H, T = 1280, 720, 50
dev = torch.device("cuda", 0)
ring = bench.device_texture_ring(W, H, 50, 0.02, 0.0, dev)
cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, 0.0)), cfg, seed=0)
eng = StepEngine(StepShape(1, T, H, W, 8 * W * H, _lib.EVS_ORDER_CANONICAL, 1000, 0.01, 100, st.uniform_thresholds), dev)
for k in range(3):
    eng.launch(ring[None], st.d_ref_log, st.d_last_event_t, t0=k * T * 1000, tick=1000)
counts, *_ = eng.fetch_info()
pool = PinnedPool(); scratch = {}
rows = [eng.ev_t, eng.ev_x, eng.ev_y, eng.ev_p]
for name in ("segments", "compact", "segments", "compact"):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        if name == "segments":
            out = d2h_segments(pool, counts, rows)
        else:
            out = d2h_compact(pool, counts, eng.info[0], rows, scratch)
        del out
    dt = (time.perf_counter() - t) / 5
    print(name, f"{dt*1e3:.2f} ms  {13*int(counts.sum())/dt/1e9:.1f} GB/s", flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
bufs = scratch["bufs"]
e0.record()
L = _lib.load()
for _ in range(10):
    L.evs_compact_segments(T, eng.info[0].data_ptr(), eng.ev_t.shape[1], *[r.data_ptr() for r in rows], *[b.data_ptr() for b in bufs], _lib.stream_ptr())
e1.record(); torch.cuda.synchronize()
print("compact kernel ms", e0.elapsed_time(e1) / 10)
