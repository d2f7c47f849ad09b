"""Diagnostic: HD T=25 fast path vs oracle over 4 steps (bench-like ring), per-segment stats."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2602_15018_b200 import _lib, events as ev
from paper_2602_15018_b200.runtime import StepEngine, StepShape
from paper_2602_15018_b200.synth import texture_frame
W, H, T = 1280, 720, 25
dev = torch.device("cuda", 0)
host = np.stack([texture_frame(W, H, 0.02 * k) for k in range(50)])
ring = torch.from_numpy(host).to(dev)
o = oracle.init_state(host[0], c_pos=0.15, c_neg=0.15, refractory_us=100, seed=0)
ref = torch.from_numpy(o.ref_log.copy()).to(dev); last = torch.from_numpy(o.last_event_t.copy()).to(dev)
eng = StepEngine(StepShape(1, T, H, W, 8 * W * H, _lib.EVS_ORDER_CANONICAL, 1000, 0.01, 100, (0.15, 0.15)), dev)
for k in range(4):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    [e.record() for e in evs]
    eng.launch(ring[(k % 2) * T:(k % 2 + 1) * T], ref, last, t0=k * T * 1000, tick=1000, stage_events=evs)
    torch.cuda.synchronize()
    counts, dropped, res, bad = eng.fetch_info()
    print(k, "stage ms", [round(evs[i].elapsed_time(evs[i + 1]), 3) for i in range(4)], flush=True)
    nbad = 0
    for f in range(T):
        fr = (k % 2) * T + f
        g = k * T + f
        ob = oracle.canonical_sort(oracle.generate(o, host[fr], g * 1000, (g + 1) * 1000, refractory_us=100))
        n = int(counts[f])
        t = eng.ev_t[f, :n].cpu().numpy()
        ok = n == len(ob) and np.array_equal(t, ob.t.astype(np.int64)) and np.array_equal(eng.ev_x[f, :n].cpu().numpy().view(np.uint16), ob.x)
        hb = np.bincount((ob.t.astype(np.int64) - g * 1000) // 8) if len(ob) else np.zeros(1, int)
        if not ok or f in (0, 24):
            print("  seg", f, "n", n, "oracle", len(ob), "ok", ok, "max bucket", hb.max(), "res", int(res[f]), ob.reservation_count, flush=True)
        nbad += not ok
    print("  bad segments", nbad, "state ok", np.array_equal(ref.cpu().numpy(), o.ref_log), np.array_equal(last.cpu().numpy(), o.last_event_t), flush=True)
