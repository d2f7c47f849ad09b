"""Per-frame fixture of the benchmark's own launch shape (bench.py self-check).

The bench workload (BASELINE configs[1]: HD 1280x720, C=0.15, refractory
100 us, 1000 us ticks, moving texture) is run here through the CPU oracle
(oracle/evsim_oracle.c, pinned against the reference by make_golden.py) for
the sequence bench.py verifies after its timed region: the 50-frame texture
ring ring[k] = _texture_frame(phase = k * 0.02) (events_bench.py:19-26),
stepped window after window (frame j of the sequence = ring[j % 50],
t_prev = 1000 j, t_now = 1000 (j + 1)), state initialised from ring[0] with
seed 0.  For every frame: event count, dropped, reservation count and the
SHA-1 of the canonical (t, x, y, p) arrays; plus the SHA-1 of the state.

    python tests/golden/make_bench_golden.py    # writes bench_hd_t50.json
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

W, H, C, REFR, TICK, DRIFT = 1280, 720, 0.15, 100, 1000, 0.02
FRAMES = 150  # one eager 50-frame step + two graph replays of one 50-frame step


def batch_sha1(t, x, y, p) -> str:
    h = hashlib.sha1()
    for a, dt in ((t, np.uint64), (x, np.uint16), (y, np.uint16), (p, np.int8)):
        h.update(np.ascontiguousarray(np.asarray(a).astype(dt, copy=False)).tobytes())
    return h.hexdigest()


def state_sha1(ref, last) -> str:
    h = hashlib.sha1()
    h.update(np.ascontiguousarray(ref, np.float32).tobytes())
    h.update(np.ascontiguousarray(last, np.int64).tobytes())
    return h.hexdigest()


def main() -> None:
    import oracle
    from paper_2602_15018_b200.synth import texture_frame

    oracle.build()
    ring = [texture_frame(W, H, k * DRIFT) for k in range(50)]
    st = oracle.init_state(ring[0], c_pos=C, c_neg=C, refractory_us=REFR, seed=0)
    frames = []
    for j in range(FRAMES):
        b = oracle.canonical_sort(oracle.generate(st, ring[j % 50], j * TICK, (j + 1) * TICK, refractory_us=REFR))
        frames.append({"count": len(b), "dropped": b.dropped_count, "reservations": b.reservation_count,
                       "sha1": batch_sha1(b.t, b.x, b.y, b.polarity)})
        if j % 10 == 0:
            print(j, len(b), flush=True)
    out = {"workload": "HD 1280x720, C=0.15, refractory 100us, 1000us ticks, texture ring of 50 frames "
                       "(phase k*0.02), seed 0, capacity 8*P", "frames": frames,
           "state_sha1": state_sha1(st.ref_log, st.last_event_t)}
    with open(os.path.join(HERE, "bench_hd_t50.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    main()
