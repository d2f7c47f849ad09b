"""The reference's chunk-parallel tests (pkg/tests/test_event_parallel.py and the
event criteria of test_acceptance.py) re-pointed at the B200 drop-in."""

import numpy as np
import pytest

from helpers import frame_from_log, random_walk_sequence

pytestmark = pytest.mark.gpu

ev = pytest.importorskip("paper_2602_15018_b200.events")


def _run_pair(frames, cfg, workers, seed=0):
    """test_event_parallel.py:113-124: state equality after every frame."""
    s_ser = ev.init_pixel_states(frames[0], cfg, seed=seed)
    s_par = s_ser.copy()
    out = []
    for k in range(1, len(frames)):
        t0, t1 = frames[k - 1].t, frames[k].t
        b_ser = ev.generate_events_serial(s_ser, frames[k], t0, t1, cfg)
        b_par = ev.generate_events_parallel(s_par, frames[k], t0, t1, cfg, workers=workers)
        out.append((b_ser, b_par))
        assert np.array_equal(s_ser.ref_log, s_par.ref_log)
        assert np.array_equal(s_ser.last_event_t, s_par.last_event_t)
    return out


def test_workers_one_matches_serial():
    for b_ser, b_par in _run_pair(random_walk_sequence(np.random.default_rng(0), 64, 48, 10), ev.EventCameraConfig(), 1):
        assert ev.canonical_sort(b_ser).same_events(ev.canonical_sort(b_par))


@pytest.mark.parametrize("workers", [2, 4, 8])
def test_multi_worker_matches_serial(workers):
    frames = random_walk_sequence(np.random.default_rng(workers), 64, 48, 8, step_std=0.15)
    for b_ser, b_par in _run_pair(frames, ev.EventCameraConfig(sigma_c=0.03), workers, seed=5):
        cs, cp = ev.canonical_sort(b_ser), ev.canonical_sort(b_par)
        assert cs.same_events(cp) and cs.dropped_count == cp.dropped_count == 0


def test_refractory_equivalence():
    frames = random_walk_sequence(np.random.default_rng(77), 32, 32, 6, step_std=0.3)
    for b_ser, b_par in _run_pair(frames, ev.EventCameraConfig(refractory_us=6000), 4):
        assert ev.canonical_sort(b_ser).same_events(ev.canonical_sort(b_par))


def test_parallel_output_is_canonical():
    frames = random_walk_sequence(np.random.default_rng(3), 48, 32, 6)
    cfg = ev.EventCameraConfig()
    st = ev.init_pixel_states(frames[0], cfg, seed=1)
    for k in range(1, len(frames)):
        b = ev.generate_events_parallel(st, frames[k], frames[k - 1].t, frames[k].t, cfg, workers=8)
        assert b.same_events(ev.canonical_sort(b))


def test_write_once_spans_disjoint_and_covering():
    frames = random_walk_sequence(np.random.default_rng(8), 64, 48, 4, step_std=0.2)
    cfg = ev.EventCameraConfig()
    st = ev.init_pixel_states(frames[0], cfg, seed=0)
    for k in range(1, len(frames)):
        stats = ev.AggregationStats(collect_spans=True)
        ev.generate_events_parallel(st, frames[k], frames[k - 1].t, frames[k].t, cfg, workers=4, stats=stats)
        covered = 0
        for base, count in sorted(stats.write_spans):
            assert base == covered
            covered += count
        assert covered == stats.events_emitted


def test_atomic_reduction_exact_64():
    """test_acceptance.py:103-112: 2048 single-event pixels -> exactly 64 chunk reservations."""
    w, h = 64, 32
    cfg = ev.EventCameraConfig()
    st = ev.init_pixel_states(frame_from_log(np.full((h, w), -2.0), 0), cfg, seed=0)
    stats = ev.AggregationStats()
    b = ev.generate_events_parallel(st, frame_from_log(np.full((h, w), -1.7), 1000), 0, 1000, cfg, workers=4,
                                    stats=stats)
    assert len(b) == w * h == 2048
    assert stats.reservation_count == (w * h) // ev.CHUNK_WIDTH == 64


def test_reservation_bound():
    frames = random_walk_sequence(np.random.default_rng(13), 40, 30, 6, step_std=0.4)
    cfg = ev.EventCameraConfig()
    st = ev.init_pixel_states(frames[0], cfg, seed=0)
    for k in range(1, len(frames)):
        stats = ev.AggregationStats()
        ev.generate_events_parallel(st, frames[k], frames[k - 1].t, frames[k].t, cfg, workers=8, stats=stats)
        assert stats.reservation_count <= -(-40 * 30 // ev.CHUNK_WIDTH) + 1


def test_bounded_capacity_counts():
    frames = random_walk_sequence(np.random.default_rng(21), 32, 24, 5, step_std=0.3)
    cap = 200
    cfg_cap = ev.EventCameraConfig(max_events_per_frame=cap)
    cfg_free = ev.EventCameraConfig(max_events_per_frame=10**9)
    s_free = ev.init_pixel_states(frames[0], cfg_free, seed=0)
    s_cap = ev.init_pixel_states(frames[0], cfg_cap, seed=0)
    for k in range(1, len(frames)):
        full = ev.generate_events_serial(s_free, frames[k], frames[k - 1].t, frames[k].t, cfg_free)
        capped = ev.generate_events_parallel(s_cap, frames[k], frames[k - 1].t, frames[k].t, cfg_cap, workers=4)
        assert len(capped) + capped.dropped_count == len(full)
        full_set = set(zip(full.t.tolist(), full.x.tolist(), full.y.tolist(), full.polarity.tolist()))
        cap_list = list(zip(capped.t.tolist(), capped.x.tolist(), capped.y.tolist(), capped.polarity.tolist()))
        assert set(cap_list) <= full_set and len(cap_list) == len(set(cap_list))
        # B200 placement is pixel-major, so the kept events are exactly the
        # serial definition's first `cap` (stronger than the reference's subset)
        first = ev.canonical_sort(ev.EventBatch(full.t[:cap], full.x[:cap], full.y[:cap], full.polarity[:cap]))
        assert capped.same_events(first)
        assert np.array_equal(s_free.ref_log, s_cap.ref_log)


def test_oracle_equivalence_acceptance_subset():
    """test_acceptance.py:79-100 (first 20 of the 100 random-walk sequences)."""
    cfg = ev.EventCameraConfig(sigma_c=0.03)
    for seq_id in range(20):
        frames = random_walk_sequence(np.random.default_rng(10_000 + seq_id), 64, 48, 50, step_std=0.08)
        s_ser = ev.init_pixel_states(frames[0], cfg, seed=seq_id)
        s_par = s_ser.copy()
        for k in range(1, len(frames)):
            t0, t1 = frames[k - 1].t, frames[k].t
            ref = ev.canonical_sort(ev.generate_events_serial(s_ser, frames[k], t0, t1, cfg))
            got = ev.generate_events_parallel(s_par, frames[k], t0, t1, cfg, workers=4)
            assert got.same_events(ref) and got.dropped_count == ref.dropped_count == 0
        assert np.array_equal(s_par.ref_log, s_ser.ref_log)


class TestCanonicalSort:  # test_event_parallel.py:82-110
    def test_empty(self):
        out = ev.canonical_sort(ev.EventBatch.empty(dropped_count=3))
        assert len(out) == 0 and out.dropped_count == 3

    def test_idempotent(self):
        b = ev.EventBatch(t=np.array([1, 1, 2], np.uint64), x=np.array([0, 1, 0], np.uint16),
                          y=np.array([0, 0, 0], np.uint16), polarity=np.array([1, -1, 1], np.int8))
        once = ev.canonical_sort(b)
        assert once.same_events(ev.canonical_sort(once))

    def test_reversed_three(self):
        b = ev.EventBatch(t=np.array([30, 20, 10], np.uint64), x=np.array([2, 1, 0], np.uint16),
                          y=np.array([2, 1, 0], np.uint16), polarity=np.array([1, 1, 1], np.int8))
        out = ev.canonical_sort(b)
        assert out.t.tolist() == [10, 20, 30] and out.x.tolist() == [0, 1, 2]

    def test_order_keys(self):
        b = ev.EventBatch(t=np.array([5, 5, 5, 5], np.uint64), x=np.array([1, 0, 0, 0], np.uint16),
                          y=np.array([0, 1, 0, 0], np.uint16), polarity=np.array([1, 1, 1, -1], np.int8))
        out = ev.canonical_sort(b)
        assert out.y.tolist() == [0, 0, 0, 1] and out.x.tolist() == [0, 0, 1, 0]
        assert out.polarity.tolist() == [-1, 1, 1, 1]


class TestHostInstrumentation:  # test_event_parallel.py:24-79 (host objects of the API)
    def test_reserve_block(self):
        cur = ev.ReservationCursor(capacity=10)
        assert ev.reserve_block(cur, 7) == (0, 7)
        assert ev.reserve_block(cur, 7) == (7, 3)
        assert ev.reserve_block(cur, 4)[1] == 0
        assert ev.reserve_block(cur, 0) == (18, 0)

    def test_chunk_mask(self):
        m = ev.compute_chunk_mask(np.array([0, 2, 1, 0, 5] + [0] * 27))
        assert m.bits == (1 << 1) | (1 << 2) | (1 << 4) and m.popcount == 3
        with pytest.raises(ValueError):
            ev.compute_chunk_mask(np.ones(33, int))
