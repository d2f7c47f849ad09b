"""CUDA path vs the CPU oracle at BASELINE.json sizes, plus golden noise / batch ops.

Exact (bit-for-bit) equality is required for event multisets, order, counts,
reservations and state; parity is checked frame by frame.
"""

import os

import numpy as np
import pytest

import oracle
from paper_2602_15018_b200.synth import texture_frame

pytestmark = pytest.mark.gpu
ev = pytest.importorskip("paper_2602_15018_b200.events")
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _sequence(W, H, frames, cfg, seed, phase0=0.0, api="parallel", drift=0.02, noise_rate=0.0):
    st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, phase0)), cfg, seed=seed)
    ost = oracle.OState(W, H, st.ref_log.copy(), st.last_event_t.copy(), st.thresholds_pos.copy(),
                        st.thresholds_neg.copy())
    cap = cfg.capacity(W, H)
    for k in range(1, frames + 1):
        vals = texture_frame(W, H, phase0 + drift * k)
        fr = ev.IntensityFrame(W, H, 1000 * k, vals)
        stats = ev.AggregationStats()
        if api == "parallel":
            got = ev.generate_events_parallel(st, fr, 1000 * (k - 1), 1000 * k, cfg, stats=stats)
        else:
            got = ev.generate_events_serial(st, fr, 1000 * (k - 1), 1000 * k, cfg)
        exp = oracle.generate(ost, vals, 1000 * (k - 1), 1000 * k, log_eps=cfg.log_eps,
                              refractory_us=cfg.refractory_us, cap=cap)
        if api == "parallel":
            assert stats.reservation_count == exp.reservation_count
            exp = oracle.canonical_sort(exp)
        assert got.same_events(exp), (W, H, k, len(got), len(exp))
        assert got.dropped_count == exp.dropped_count
        assert np.array_equal(st.ref_log, ost.ref_log)
        assert np.array_equal(st.last_event_t, ost.last_event_t)


def test_config1_davis_texture():
    _sequence(346, 260, 40, ev.EventCameraConfig(max_events_per_frame=32 * 346 * 260), seed=0)


def test_config2_hd_refractory():
    _sequence(1280, 720, 4, ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100), seed=0)


def test_config3_vga_stream():
    _sequence(640, 480, 4, ev.EventCameraConfig(), seed=5, phase0=0.137 * 5)


def test_config4_fhd_multicrossing_serial_order():
    _sequence(1920, 1080, 2, ev.EventCameraConfig(c_pos=0.05, c_neg=0.05), seed=1, api="serial")


def test_sigma_refractory_large_steps():
    cfg = ev.EventCameraConfig(c_pos=0.1, c_neg=0.12, sigma_c=0.03, refractory_us=300)
    _sequence(333, 211, 8, cfg, seed=9, drift=0.11)


def test_capacity_overflow_large_frame():
    cfg = ev.EventCameraConfig(c_pos=0.05, c_neg=0.05, max_events_per_frame=100_000)
    _sequence(640, 480, 3, cfg, seed=2)


@pytest.mark.parametrize("W,H,api", [(65535, 3, "parallel"), (3, 65535, "parallel"), (65535, 2, "serial"),
                                      (1, 1, "parallel"), (31, 1, "serial")])
def test_extreme_shapes(W, H, api):
    """Coordinates at the 16-bit limits of the packed keys (x or y = 65534),
    one-pixel and one-row sensors."""
    _sequence(W, H, 3, ev.EventCameraConfig(c_pos=0.1, c_neg=0.1, refractory_us=50), seed=3, api=api,
              drift=0.07)


def test_noise_golden():
    g = dict(np.load(os.path.join(GOLD, "noise.npz")))
    i = 0
    while f"case{i}" in g:
        w, h, t0, t1, seed = [int(v) for v in g[f"case{i}"]]
        b = ev.inject_noise_events(w, h, t0, t1, float(g[f"rate{i}"][0]), seed)
        assert np.array_equal(b.t.astype(np.int64), g[f"t{i}"]), i
        assert np.array_equal(b.x, g[f"x{i}"]) and np.array_equal(b.y, g[f"y{i}"])
        assert np.array_equal(b.polarity, g[f"p{i}"])
        i += 1


@pytest.mark.parametrize("W,H,dt,rate,seed", [
    (1920, 1080, 1000, 10.0, 11),      # config 4 rate
    (346, 260, 1000, 2000.0, 5),       # lam = 2
    (64, 48, 1000, 9500.0, 3),         # lam = 9.5, long multiplication runs
    (96, 64, 1000, 10000.0, 8),        # lam = 10 -> PTRS
    (40, 30, 1000, 60000.0, 2**64 - 5),
    (1, 1, 1000, 50.0, 0),
])
def test_noise_vs_oracle(W, H, dt, rate, seed):
    b = ev.inject_noise_events(W, H, 0, dt, rate, seed)
    o = oracle.noise(W, H, 0, dt, rate, seed)
    assert b.same_events(o)


def test_batch_ops_golden():
    g = dict(np.load(os.path.join(GOLD, "batch_ops.npz")))
    b = ev.EventBatch(g["t"].astype(np.uint64), g["x"], g["y"], g["p"], dropped_count=4)
    assert np.array_equal(ev.accumulate_events_to_image(b, 1500, 2500, 40, 30), g["acc"])
    cs = ev.canonical_sort(b)
    lb = ev.limit_bandwidth(cs, 2.0e6, 100)
    assert np.array_equal(lb.t.astype(np.int64), g["lb_t"]) and np.array_equal(lb.x, g["lb_x"])
    assert lb.dropped_count == int(g["lb_dropped"][0])


def test_large_batch_ops_vs_oracle():
    from paper_2602_15018_b200.represent import voxel_grid

    rng = np.random.default_rng(4)
    n = 1_000_003
    b = ev.EventBatch(t=rng.integers(5000, 25000, n).astype(np.uint64), x=rng.integers(0, 346, n).astype(np.uint16),
                      y=rng.integers(0, 260, n).astype(np.uint16),
                      polarity=(rng.integers(0, 2, n) * 2 - 1).astype(np.int8))
    ob = oracle.OBatch(b.t, b.x, b.y, b.polarity)
    cs = ev.canonical_sort(b)
    assert cs.same_events(oracle.canonical_sort(ob))
    assert np.array_equal(ev.accumulate_events_to_image(b, 7000, 20000, 346, 260),
                          oracle.accumulate(ob, 7000, 20000, 346, 260))
    np.testing.assert_array_equal(voxel_grid(b, 5000, 25000, 346, 260, bins=5),
                                  oracle.voxel(ob, 5000, 25000, 5, 346, 260))
    lb = ev.limit_bandwidth(cs, 3.3e7, 137)
    olb = oracle.limit_bandwidth(oracle.canonical_sort(ob), 3.3e7, 137)
    assert lb.same_events(olb) and lb.dropped_count == olb.dropped_count


def test_canonical_sort_general_golden():
    """canonical_sort of a batch outside the simulator's range (uint64 times
    spanning > 2^31 us and >= 2^63, any int8 polarity) equals the reference's
    lexsort (tests/golden/sort_general.npz, made by the reference itself)."""
    g = dict(np.load(os.path.join(GOLD, "sort_general.npz")))
    b = ev.EventBatch(g["t"].view(np.uint64), g["x"], g["y"], g["p"], dropped_count=9)
    cs = ev.canonical_sort(b)
    assert np.array_equal(cs.t.view(np.int64), g["cs_t"]) and np.array_equal(cs.x, g["cs_x"])
    assert np.array_equal(cs.y, g["cs_y"]) and np.array_equal(cs.polarity, g["cs_p"])
    assert cs.dropped_count == 9
    # a batch only slightly outside (t-span 2^31) and a large random one vs the oracle
    rng = np.random.default_rng(8)
    for n, span in ((70_001, 1 << 31), (1_500_000, 1 << 45)):
        b = ev.EventBatch(t=rng.integers(10, 10 + span, n).astype(np.uint64),
                          x=rng.integers(0, 64, n).astype(np.uint16), y=rng.integers(0, 48, n).astype(np.uint16),
                          polarity=rng.integers(-3, 3, n).astype(np.int8))
        assert ev.canonical_sort(b).same_events(oracle.canonical_sort(oracle.OBatch(b.t, b.x, b.y, b.polarity)))
