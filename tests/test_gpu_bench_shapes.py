"""Parity at the shapes the numbers are measured on (BASELINE configs 1-5).

Every test drives the CUDA path the way bench.py / tools/bench_configs.py do
(same launch shapes: frames per call, streams per call, K1 frame chunking,
K2 group sizes, fused validation, CUDA-graph replay with the device clock)
and compares every frame bit for bit with the CPU oracle (events, order,
counts, dropped, reservation counts, state).  The oracle is pinned against
the reference by tests/golden/make_golden.py.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle
from paper_2602_15018_b200 import _lib
from paper_2602_15018_b200 import events as ev
from paper_2602_15018_b200.synth import texture_frame

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _seg_arrays(eng, g, n):
    return (eng.ev_t[g, :n].cpu().numpy(), eng.ev_x[g, :n].cpu().numpy().view(np.uint16),
            eng.ev_y[g, :n].cpu().numpy().view(np.uint16), eng.ev_p[g, :n].cpu().numpy())


def _same_segment(eng, g, counts, dropped, res, ob, ctx):
    n = int(counts[g])
    assert n == len(ob), (ctx, n, len(ob))
    t, x, y, p = _seg_arrays(eng, g, n)
    assert np.array_equal(t, ob.t.astype(np.int64)), ctx
    assert np.array_equal(x, ob.x) and np.array_equal(y, ob.y), ctx
    assert np.array_equal(p, ob.polarity), ctx
    assert int(dropped[g]) == ob.dropped_count, ctx
    assert int(res[g]) == ob.reservation_count, ctx


def test_hd_t50_graph_replay_matches_oracle():
    """(i) bench.py's launch shape: HD, C=0.15, refractory 100 us, T=50 frames
    per evs_step, capacity 8P, validation fused into K1 (6 chunks of 9 frames
    per tile, chunk hand-offs), K2 groups of 16 tiles; one eager step then two
    replays of the captured graph (device clock) = 150 frames vs the oracle."""
    import torch

    from paper_2602_15018_b200.runtime import StepEngine, StepShape

    import bench

    W, H, T, C, REFR, TICK = 1280, 720, 50, 0.15, 100, 1000
    P = W * H
    dev = torch.device("cuda")
    ring = bench.device_texture_ring(W, H, T, 0.02, 0.0, dev)
    host_ring = ring.cpu().numpy()
    cfg = ev.EventCameraConfig(c_pos=C, c_neg=C, refractory_us=REFR)
    st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, 0.0)), cfg, seed=0)
    eng = StepEngine(StepShape(1, T, H, W, 8 * P, _lib.EVS_ORDER_CANONICAL, TICK, cfg.log_eps, REFR,
                               st.uniform_thresholds), dev)
    ost = oracle.init_state(host_ring[0], c_pos=C, c_neg=C, refractory_us=REFR, seed=0)
    for i in range(3):
        if i == 0:
            eng.launch(ring, st.d_ref_log, st.d_last_event_t, t0=0, tick=TICK, validate=True)
        else:
            if i == 1:
                eng.capture([ring], st.d_ref_log, st.d_last_event_t, tick=TICK, t0=T * TICK)
            eng.replay()
        torch.cuda.synchronize()
        counts, dropped, res, bad = eng.fetch_info()
        assert bad == _lib.NO_BAD
        for f in range(T):
            j = i * T + f
            ob = oracle.canonical_sort(oracle.generate(ost, host_ring[f], j * TICK, (j + 1) * TICK,
                                                       refractory_us=REFR))
            _same_segment(eng, f, counts, dropped, res, ob, (i, f))
        assert np.array_equal(st.d_ref_log.cpu().numpy(), ost.ref_log)
        assert np.array_equal(st.d_last_event_t.cpu().numpy(), ost.last_event_t)


def test_bench_self_check_fixture():
    """bench.py's own self-check (verify_launch_shape) passes against the
    committed oracle fixture tests/golden/bench_hd_t50.json."""
    import torch

    import bench

    assert bench.verify_launch_shape(torch.device("cuda"), 50) == []
    assert bench.verify_launch_shape(torch.device("cuda"), 50, pipelined=True) == []


def _sim_run(W, H, S, T, c, refr, steps, cap=None, noise_hz=0.0, canonical=True):
    """EventSimulator over `steps` steps of moving texture (stream s at phase
    0.137 s + 0.02 k, seed s), every (stream, frame) compared with the oracle;
    yields (sim, oracle states, step index) after each verified step."""
    import torch

    from paper_2602_15018_b200.simulator import EventSimulator

    cfg = ev.EventCameraConfig(c_pos=c, c_neg=c, refractory_us=refr, noise_rate_hz=noise_hz,
                               max_events_per_frame=cap)
    sim = EventSimulator(W, H, streams=S, frames_per_step=T, config=cfg, canonical=canonical)
    f0 = [texture_frame(W, H, 0.137 * s) for s in range(S)]
    sim.reset(f0, seeds=list(range(S)))
    ost = [oracle.init_state(f0[s], c_pos=c, c_neg=c, refractory_us=refr, seed=s) for s in range(S)]
    capv = cfg.capacity(W, H)
    for i in range(steps):
        obs = [[None] * T for _ in range(S)]
        frames = np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (i * T + f + 1)) for f in range(T)]
                           for s in range(S)])
        sim.step(torch.from_numpy(frames).cuda())
        r = sim.result()
        counts = r.counts.ravel()
        dropped = r.dropped.ravel()
        res = r.reservations.ravel()
        for s in range(S):
            for f in range(T):
                k = i * T + f
                ob = oracle.generate(ost[s], frames[s, f], k * 1000, (k + 1) * 1000, refractory_us=refr, cap=capv)
                obs[s][f] = ob
                if canonical:
                    ob = oracle.canonical_sort(ob)
                _same_segment(sim.engine, s * T + f, counts, dropped, res, ob, (i, s, f))
        yield sim, ost, obs, i
    for s in range(S):
        assert np.array_equal(sim.ref[s].cpu().numpy(), ost[s].ref_log)
        assert np.array_equal(sim.last[s].cpu().numpy(), ost[s].last_event_t)


def test_config1_davis_1000_frames():
    """(ii) config 1: DAVIS 346x260, C=0.2, capacity 32 P (events_bench.py:40),
    1000 frames as 20 steps of T=50, every frame and the state vs the oracle."""
    for sim, ost, _, i in _sim_run(346, 260, 1, 50, 0.2, 0, 20, cap=32 * 346 * 260):
        assert np.array_equal(sim.ref[0].cpu().numpy(), ost[0].ref_log), i


def test_config3_64_vga_streams():
    """(iii) config 3: 64 independent 640x480 cameras in one call (S=64, T=4), 2 steps."""
    for _ in _sim_run(640, 480, 64, 4, 0.2, 0, 2):
        pass


def test_config5_256_davis_streams_with_histograms():
    """(iv) config 5: 256 DAVIS streams per call (S=256, T=4) plus the signed
    histograms of every stream (evs_step_histogram, model.py:249-262)."""
    W, H, S, T = 346, 260, 256, 4
    for sim, ost, obs, i in _sim_run(W, H, S, T, 0.2, 0, 1):
        pass
    t_end = T * 1000
    for window, t_end in ((T * 1000, T * 1000), (1500, 2500)):
        got = sim.histograms(window, t_end).cpu().numpy()
        for s in range(S):
            b = oracle.concat(obs[s])
            assert np.array_equal(got[s], oracle.accumulate(b, window, t_end, W, H)), (window, s)


def test_config4_1080p_voxel_window_with_noise():
    """(v) config 4: 1920x1080, C=0.05 (multi-crossing, up to 5 per pixel-frame),
    T=20 frames per call, 10 Hz exact noise per frame, 5-bin voxel grid of the
    20-frame window (EventSimulator.voxel_window) vs the oracle's voxel grid of
    the concatenated signal + noise batch; the first frames' canonical events
    and every frame's counts vs the oracle."""
    import torch

    from paper_2602_15018_b200.simulator import EventSimulator, mix64

    W, H, T, C = 1920, 1080, 20, 0.05
    cfg = ev.EventCameraConfig(c_pos=C, c_neg=C, noise_rate_hz=10.0)
    sim = EventSimulator(W, H, streams=1, frames_per_step=T, config=cfg)
    f0 = texture_frame(W, H, 0.0)
    sim.reset([f0], seeds=[0])
    ost = oracle.init_state(f0, c_pos=C, c_neg=C, seed=0)
    frames = np.stack([[texture_frame(W, H, 0.02 * (f + 1)) for f in range(T)]])
    sim.step(torch.from_numpy(frames).cuda())
    r = sim.result()
    seeds = [mix64(0, 0x6E6F6973, f) for f in range(T)]
    parts = []
    for f in range(T):
        ob = oracle.generate(ost, frames[0, f], f * 1000, (f + 1) * 1000)
        assert int(r.counts[0, f]) == len(ob) and int(r.dropped[0, f]) == ob.dropped_count, f
        assert int(r.reservations[0, f]) == ob.reservation_count, f
        if f < 3:
            _same_segment(sim.engine, f, r.counts.ravel(), r.dropped.ravel(), r.reservations.ravel(),
                          oracle.canonical_sort(ob), f)
        parts.append(ob)
        parts.append(oracle.noise(W, H, f * 1000, (f + 1) * 1000, cfg.noise_rate_hz, seeds[f]))
    assert np.bincount(parts[0].y.astype(np.int64) * W + parts[0].x).max() >= 3  # multi-crossing
    exp = oracle.voxel(oracle.concat(parts), 0, T * 1000, 5, W, H)
    got = sim.voxel_window(0, bins=5, noise_seeds=seeds).cpu().numpy()
    np.testing.assert_array_equal(got, exp)
    assert np.array_equal(sim.ref[0].cpu().numpy(), ost.ref_log)
    assert np.array_equal(sim.last[0].cpu().numpy(), ost.last_event_t)


def test_acceptance_100_sequences_vs_oracle():
    """(vi) test_acceptance.py:79-100: all 100 random-walk sequences (64x48, 50
    frames, sigma_c=0.03, seeds 10000+i), both drop-in entry points, every frame
    vs the oracle (serial: pixel-major; parallel: canonical), and the state."""
    from helpers import random_walk_sequence

    cfg = ev.EventCameraConfig(sigma_c=0.03)
    for seq_id in range(100):
        frames = random_walk_sequence(np.random.default_rng(10_000 + seq_id), 64, 48, 50, step_std=0.08)
        s_ser = ev.init_pixel_states(frames[0], cfg, seed=seq_id)
        s_par = s_ser.copy()
        ost = oracle.init_state(frames[0].values, sigma_c=0.03, seed=seq_id)
        assert np.array_equal(s_ser.thresholds_pos, ost.thresholds_pos)
        for k in range(1, len(frames)):
            t0, t1 = frames[k - 1].t, frames[k].t
            ob = oracle.generate(ost, frames[k].values, t0, t1)
            a = ev.generate_events_serial(s_ser, frames[k], t0, t1, cfg)
            b = ev.generate_events_parallel(s_par, frames[k], t0, t1, cfg, workers=4)
            assert a.same_events(ob) and a.dropped_count == ob.dropped_count == 0, (seq_id, k)
            assert b.same_events(oracle.canonical_sort(ob)), (seq_id, k)
        assert np.array_equal(s_ser.ref_log, ost.ref_log) and np.array_equal(s_par.ref_log, ost.ref_log)
        assert np.array_equal(s_par.last_event_t, ost.last_event_t)


@pytest.mark.parametrize("W,H,order,refr", [(1280, 720, 1, 100), (640, 480, 0, 0)])
def test_pipelined_one_frame_steps_match_oracle(W, H, order, refr):
    """runtime.PipelinedSteps (bench.py's per-frame rate): one-frame steps on two
    engines / streams, step i+1 waiting only for step i's K1, replayed as one
    graph; every frame's events (canonical or pixel-major) and the state vs
    the oracle."""
    import torch

    from paper_2602_15018_b200.runtime import PipelinedSteps, StepShape

    import bench

    P, TICK = W * H, 1000
    dev = torch.device("cuda")
    ring = bench.device_texture_ring(W, H, 50, 0.02, 0.0, dev)
    host = ring.cpu().numpy()
    cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=refr)
    st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, 0.0)), cfg, seed=0)
    ost = oracle.init_state(host[0], c_pos=0.15, c_neg=0.15, refractory_us=refr, seed=0)
    pipe = PipelinedSteps(StepShape(1, 1, H, W, 8 * P, order, TICK, cfg.log_eps, refr, st.uniform_thresholds), dev)
    k = 0
    for e in pipe.engines:  # an eager step on each engine first (as bench.py does)
        e.launch(ring[k:k + 1], st.d_ref_log, st.d_last_event_t, t0=k * TICK, tick=TICK)
        ob = oracle.generate(ost, host[k], k * TICK, (k + 1) * TICK, refractory_us=refr)
        k += 1
    pipe.capture([ring[k:k + 1], ring[k + 1:k + 2]], st.d_ref_log, st.d_last_event_t, tick=TICK, t0=k * TICK)
    for rep in range(3):
        pipe.replay()
        torch.cuda.synchronize()
        for j, e in enumerate(pipe.engines):  # the graph's frames are always ring[2] and ring[3]
            counts, dropped, res, bad = e.fetch_info()
            assert bad == _lib.NO_BAD
            ob = oracle.generate(ost, host[2 + j], k * TICK, (k + 1) * TICK, refractory_us=refr)
            if order == 1:
                ob = oracle.canonical_sort(ob)
            _same_segment(e, 0, counts, dropped, res, ob, (rep, j))
            k += 1
        assert np.array_equal(st.d_ref_log.cpu().numpy(), ost.ref_log)
        assert np.array_equal(st.d_last_event_t.cpu().numpy(), ost.last_event_t)
