"""Diagnostic: tile-order path vs oracle on the engine test case, first mismatches."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2602_15018_b200 import _lib
from paper_2602_15018_b200.runtime import StepEngine, StepShape
from paper_2602_15018_b200.synth import texture_frame
S, T, H, W, refr = 1, 4, 90, 160, 100
frames = np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (k + 1)) for k in range(T)] for s in range(S)])
o = oracle.init_state(texture_frame(W, H, 0.0), c_pos=0.15, c_neg=0.15, refractory_us=refr, seed=0)
dev = torch.device("cuda")
ref = torch.from_numpy(o.ref_log[None].copy()).to(dev); last = torch.from_numpy(o.last_event_t[None].copy()).to(dev)
eng = StepEngine(StepShape(S, T, H, W, 8 * H * W, 1, 1000, 0.01, refr, (0.15, 0.15)), dev)
eng.launch(torch.from_numpy(frames).to(dev), ref, last, t0=0, tick=1000)
counts, dropped, res, bad = eng.fetch_info()
for f in range(T):
    ob = oracle.generate(o, frames[0, f], f * 1000, (f + 1) * 1000, refractory_us=refr)
    n = int(counts[f])
    t = eng.ev_t[f, :n].cpu().numpy(); x = eng.ev_x[f, :n].cpu().numpy().view(np.uint16); y = eng.ev_y[f, :n].cpu().numpy().view(np.uint16)
    exp = oracle.canonical_sort(ob)
    gs = set(zip(t.tolist(), x.tolist(), y.tolist())); es = set(zip(exp.t.astype(np.int64).tolist(), exp.x.tolist(), exp.y.tolist()))
    print("frame", f, "n", n, "oracle", len(exp), "missing", sorted(es - gs)[:8], "extra", sorted(gs - es)[:8])
