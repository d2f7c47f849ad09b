"""Generate golden vectors by running the REFERENCE itself (evsim, Python/numpy).

Run in the authoring container (the reference exists only here):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports /root/reference/pkg/src/evsim read-only and writes compressed
.npz fixtures next to this file.  The GPU box never reads /root/reference;
tests compare the oracle and the CUDA path against these files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    from evsim.bench.events_bench import _texture_frame
    from evsim.events import (
        AggregationStats,
        EventCameraConfig,
        accumulate_events_to_image,
        canonical_sort,
        generate_events_parallel,
        generate_events_serial,
        init_pixel_states,
        inject_noise_events,
        limit_bandwidth,
    )
    from evsim.events.types import EventBatch
    from evsim.sim.orchestrator import _mix64
    from helpers import random_walk_sequence

    def seq_case(name, frames_vals, times, cfg, seed, serial=True):
        """Run the reference over a frame sequence; store inputs, per-frame events, states."""
        from evsim.events.types import IntensityFrame

        h, w = frames_vals[0].shape
        f0 = IntensityFrame(width=w, height=h, t=int(times[0]), values=frames_vals[0])
        st = init_pixel_states(f0, cfg, seed=seed)
        out = {
            "frames": np.stack(frames_vals).astype(np.float32),
            "times": np.asarray(times, np.int64),
            "thp": st.thresholds_pos.copy(), "thn": st.thresholds_neg.copy(),
            "ref0": st.ref_log.copy(), "last0": st.last_event_t.copy(),
            "cfg": np.array([cfg.c_pos, cfg.c_neg, cfg.sigma_c, cfg.refractory_us, cfg.log_eps,
                             cfg.capacity(w, h)], np.float64),
        }
        ev_t, ev_x, ev_y, ev_p, ev_n, drops, res, refs, lasts = [], [], [], [], [], [], [], [], []
        for k in range(1, len(frames_vals)):
            fr = IntensityFrame(width=w, height=h, t=int(times[k]), values=frames_vals[k])
            if serial:
                b = generate_events_serial(st, fr, int(times[k - 1]), int(times[k]), cfg)
                stats = None
            else:
                stats = AggregationStats()
                b = generate_events_parallel(st, fr, int(times[k - 1]), int(times[k]), cfg,
                                             workers=1, stats=stats)
                b = canonical_sort(b)
            ev_t.append(b.t.astype(np.int64)); ev_x.append(b.x); ev_y.append(b.y)
            ev_p.append(b.polarity); ev_n.append(len(b)); drops.append(b.dropped_count)
            res.append(stats.reservation_count if stats else -1)
            refs.append(st.ref_log.copy()); lasts.append(st.last_event_t.copy())
        out.update(ev_t=np.concatenate(ev_t), ev_x=np.concatenate(ev_x), ev_y=np.concatenate(ev_y),
                   ev_p=np.concatenate(ev_p), ev_n=np.array(ev_n, np.int64),
                   dropped=np.array(drops, np.int64), res=np.array(res, np.int64),
                   refs=np.stack(refs), lasts=np.stack(lasts), serial=np.array(serial))
        np.savez_compressed(os.path.join(HERE, f"gen_{name}.npz"), **out)
        print(name, "events/frame", ev_n[:5], "...")

    # 1) DAVIS texture, C=0.2 (config 1 shape), serial order, 4 frames
    W, H = 346, 260
    tex = [_texture_frame(W, H, k * 0.02, k * 1000).values for k in range(0, 5)]
    seq_case("texture_davis", tex, [k * 1000 for k in range(5)],
             EventCameraConfig(max_events_per_frame=32 * W * H), seed=0, serial=True)
    # 2) HD-like refractory texture crop (C=0.15, refr 100) canonical order via parallel
    W2, H2 = 160, 90
    tex2 = [_texture_frame(W2, H2, k * 0.02, k * 1000).values for k in range(0, 5)]
    seq_case("texture_refr_canon", tex2, [k * 1000 for k in range(5)],
             EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100), seed=1, serial=False)
    # 3) acceptance-style random walk with sigma_c (test_acceptance.py:79-100)
    rng = np.random.default_rng(10_000)
    frs = random_walk_sequence(rng, 64, 48, 12, step_std=0.08)
    seq_case("walk_sigma", [f.values for f in frs], [f.t for f in frs],
             EventCameraConfig(sigma_c=0.03), seed=0, serial=True)
    # 4) refractory random walk (test_event_parallel.py:144-149)
    rng = np.random.default_rng(77)
    frs = random_walk_sequence(rng, 32, 32, 6, step_std=0.3)
    seq_case("walk_refr", [f.values for f in frs], [f.t for f in frs],
             EventCameraConfig(refractory_us=6000), seed=0, serial=True)
    # 5) bounded capacity (test_event_parallel.py:208-229)
    rng = np.random.default_rng(21)
    frs = random_walk_sequence(rng, 32, 24, 5, step_std=0.3)
    seq_case("walk_cap", [f.values for f in frs], [f.t for f in frs],
             EventCameraConfig(max_events_per_frame=200), seed=0, serial=True)
    # 6) multi-crossing: large steps, C=0.05, dt=10000
    rng = np.random.default_rng(5)
    frs = random_walk_sequence(rng, 40, 30, 6, step_std=0.4)
    seq_case("walk_multi", [f.values for f in frs], [f.t for f in frs],
             EventCameraConfig(c_pos=0.05, c_neg=0.07, refractory_us=50), seed=3, serial=True)

    # noise (model.py:174-212), including PTRS (lam >= 10) and orchestrator seeds
    noise = {}
    cases = [(10, 10, 0, 1000, 100.0, 0), (100, 100, 0, 1_000_000, 10.0, 42),
             (4, 4, 0, 1_000_000, 500.0, 1), (20, 20, 0, 50000, 100.0, 7),
             (64, 48, 1000, 2000, 3000.0, _mix64(5, 0x6E6F6973, 3)),
             (346, 260, 0, 1000, 10.0, _mix64(0, 0x6E6F6973, 0)),
             (64, 48, 0, 1000, 2500.0, 2**40 + 17)]
    for i, (w, h, t0, t1, rate, seed) in enumerate(cases):
        b = inject_noise_events(w, h, t0, t1, rate, seed)
        noise[f"case{i}"] = np.array([w, h, t0, t1, seed], np.uint64)
        noise[f"rate{i}"] = np.array([rate])
        noise[f"t{i}"] = b.t.astype(np.int64)
        noise[f"x{i}"] = b.x
        noise[f"y{i}"] = b.y
        noise[f"p{i}"] = b.polarity
    np.savez_compressed(os.path.join(HERE, "noise.npz"), **noise)

    # canonical sort, accumulation, bandwidth limit on a random batch
    rng = np.random.default_rng(123)
    n = 5000
    b = EventBatch(t=rng.integers(0, 3000, n).astype(np.uint64), x=rng.integers(0, 40, n).astype(np.uint16),
                   y=rng.integers(0, 30, n).astype(np.uint16),
                   polarity=(rng.integers(0, 2, n) * 2 - 1).astype(np.int8), dropped_count=4)
    cs = canonical_sort(b)
    acc = accumulate_events_to_image(b, 1500, 2500, 40, 30)
    lb = limit_bandwidth(cs, 2.0e6, 100)
    np.savez_compressed(os.path.join(HERE, "batch_ops.npz"),
                        t=b.t.astype(np.int64), x=b.x, y=b.y, p=b.polarity,
                        cs_t=cs.t.astype(np.int64), cs_x=cs.x, cs_y=cs.y, cs_p=cs.polarity,
                        acc=acc, lb_t=lb.t.astype(np.int64), lb_x=lb.x, lb_y=lb.y, lb_p=lb.polarity,
                        lb_dropped=np.array([lb.dropped_count]))

    # PCG64 states for seeds (numpy SeedSequence)
    seeds = [0, 1, 42, 12345, 2**32 - 1, 2**32, 2**63 + 5, _mix64(7, 0x6E6F6973, 11), 2**64 - 1]
    states = []
    for s in seeds:
        st = np.random.PCG64(s).state["state"]
        states.append([st["state"] >> 64, st["state"] & (2**64 - 1), st["inc"] >> 64, st["inc"] & (2**64 - 1)])
    draws = np.random.default_rng(99).integers(0, 2**64, 64, dtype=np.uint64, endpoint=False)
    raw = np.random.PCG64(99).random_raw(64)
    np.savez_compressed(os.path.join(HERE, "pcg64.npz"), seeds=np.array(seeds, dtype=object).astype(str),
                        states=np.array(states, np.uint64), raw99=raw, ints99=draws)
    sort_general()
    print("golden fixtures written to", HERE)


def sort_general() -> None:
    """canonical_sort (parallel.py:112-123) of a batch outside the simulator's
    range: uint64 times spanning > 2^31 us and >= 2^63, any int8 polarity,
    duplicate (t, y, x) with different polarities."""
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from evsim.events import canonical_sort
    from evsim.events.types import EventBatch

    rng = np.random.default_rng(321)
    n = 20000
    t = np.concatenate([rng.integers(0, 2**40, n // 4, dtype=np.uint64),
                        rng.integers(2**63 - 50, 2**63 + 50, n // 4, dtype=np.uint64),
                        rng.integers(0, 40, n // 4, dtype=np.uint64),
                        rng.integers(2**64 - 2**33, 2**64 - 1, n - 3 * (n // 4), dtype=np.uint64,
                                     endpoint=True)])
    x = rng.integers(0, 7, n).astype(np.uint16)
    y = rng.integers(0, 5, n).astype(np.uint16)
    x[: n // 8] = rng.integers(0, 65536, n // 8)
    p = rng.integers(-128, 128, n).astype(np.int8)
    p[n // 2:] = (rng.integers(0, 2, n - n // 2) * 2 - 1)
    b = EventBatch(t=t, x=x, y=y, polarity=p, dropped_count=9)
    cs = canonical_sort(b)
    np.savez_compressed(os.path.join(HERE, "sort_general.npz"), t=t.view(np.int64), x=x, y=y, p=p,
                        cs_t=cs.t.view(np.int64), cs_x=cs.x, cs_y=cs.y, cs_p=cs.polarity)


if __name__ == "__main__":
    if sys.argv[1:] == ["sort_general"]:
        sort_general()
    else:
        main()
