"""Batched EventSimulator (S streams x T frames, device resident) and the
SimNode tick flow (generate -> noise -> concat -> canonical_sort,
orchestrator.py:159-172) against the CPU oracle."""

import numpy as np
import pytest

import oracle
from paper_2602_15018_b200.synth import texture_frame

pytestmark = pytest.mark.gpu
ev = pytest.importorskip("paper_2602_15018_b200.events")


def test_simnode_tick_flow_with_noise_matches_oracle():
    W, H, seed = 160, 90, 42
    cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100, noise_rate_hz=300.0)
    st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, 0.0)), cfg,
                              seed=oracle.mix64(seed, 0x70697865))
    ost = oracle.OState(W, H, st.ref_log.copy(), st.last_event_t.copy(), st.thresholds_pos.copy(),
                        st.thresholds_neg.copy())
    for k in range(5):
        t_prev, t_now = k * 1000, (k + 1) * 1000
        vals = texture_frame(W, H, 0.02 * (k + 1))
        sig = ev.generate_events_parallel(st, ev.IntensityFrame(W, H, t_now, vals), t_prev, t_now, cfg)
        nz = ev.inject_noise_events(W, H, t_prev, t_now, cfg.noise_rate_hz, seed=oracle.mix64(seed, 0x6E6F6973, k))
        got = ev.canonical_sort(ev.concat_batches([sig, nz]))
        o_sig = oracle.generate(ost, vals, t_prev, t_now, refractory_us=100)
        o_nz = oracle.noise(W, H, t_prev, t_now, cfg.noise_rate_hz, oracle.mix64(seed, 0x6E6F6973, k))
        exp = oracle.canonical_sort(oracle.concat([o_sig, o_nz]))
        assert len(nz) > 0
        assert got.same_events(exp) and got.dropped_count == exp.dropped_count


def test_simulator_streams_frames_noise_and_representations():
    import torch

    from paper_2602_15018_b200.simulator import EventSimulator, mix64

    S, T, W, H = 3, 2, 128, 72
    cfg = ev.EventCameraConfig(c_pos=0.1, c_neg=0.1, refractory_us=50, noise_rate_hz=500.0)
    sim = EventSimulator(W, H, streams=S, frames_per_step=T, config=cfg)
    f0 = [texture_frame(W, H, 0.137 * s) for s in range(S)]
    sim.reset(f0, seeds=[10 + s for s in range(S)])
    ost = [oracle.init_state(f0[s], c_pos=0.1, c_neg=0.1, refractory_us=50, seed=10 + s) for s in range(S)]
    k = 0
    for step in range(3):
        frames = np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (k + f + 1)) for f in range(T)] for s in range(S)])
        sim.step(torch.from_numpy(frames).cuda())
        res = sim.result()
        for s in range(S):
            for f in range(T):
                t_prev, t_now = (k + f) * 1000, (k + f + 1) * 1000
                o_sig = oracle.generate(ost[s], frames[s, f], t_prev, t_now, refractory_us=50)
                assert res.counts[s, f] == len(o_sig) and res.reservations[s, f] == o_sig.reservation_count
                nseed = mix64(99 + s, 0x6E6F6973, k + f)
                got = sim.segment_with_noise(s, f, nseed).to_host()
                o_nz = oracle.noise(W, H, t_prev, t_now, 500.0, nseed)
                exp = oracle.canonical_sort(oracle.concat([o_sig, o_nz]))
                assert got.same_events(exp), (step, s, f)
                if f == T - 1:
                    hist = sim.histogram(sim.segment(s, f), 1000, t_now).cpu().numpy()
                    assert np.array_equal(hist, oracle.accumulate(o_sig, 1000, t_now, W, H))
                    vox = sim.voxel(sim.segment(s, f), t_prev, t_now, bins=5).cpu().numpy()
                    np.testing.assert_array_equal(vox, oracle.voxel(o_sig, t_prev, t_now, 5, W, H))
            assert np.array_equal(sim.ref[s].cpu().numpy(), ost[s].ref_log)
        k += T


def test_simulator_graph_replay_multistream():
    import torch

    from paper_2602_15018_b200.simulator import EventSimulator

    S, W, H = 4, 96, 64
    cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
    sim = EventSimulator(W, H, streams=S, frames_per_step=1, config=cfg)
    f0 = [texture_frame(W, H, 0.137 * s) for s in range(S)]
    sim.reset(f0)
    ost = [oracle.init_state(f0[s], c_pos=0.15, c_neg=0.15, refractory_us=100, seed=s) for s in range(S)]
    ring = torch.from_numpy(np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (i + 1)) for s in range(S)]
                                      for i in range(5)])).cuda()  # [5, S, H, W]
    sim.step(ring[0])  # eager first step
    sim.result()
    for s in range(S):
        oracle.generate(ost[s], ring[0, s].cpu().numpy(), 0, 1000, refractory_us=100)
    windows = [ring[i].unsqueeze(1).contiguous() for i in range(1, 5)]
    sim.capture(windows)
    t = 1000
    for _rep in range(2):
        sim.replay()
        res = sim.result()
        for i in range(1, 5):
            for s in range(S):
                o = oracle.generate(ost[s], ring[i, s].cpu().numpy(), t, t + 1000, refractory_us=100)
                if i == 4:
                    assert res.counts[s, 0] == len(o)
                    assert sim.segment(s, 0).to_host().same_events(oracle.canonical_sort(o))
            t += 1000
        for s in range(S):
            assert np.array_equal(sim.ref[s].cpu().numpy(), ost[s].ref_log)


def test_step_host_matches_oracle():
    """Host buffers in / host EventBatch out (EventSimulator.step_host), S x T batch."""
    import numpy as np

    from paper_2602_15018_b200.simulator import EventSimulator

    S, T, H, W = 3, 4, 40, 56
    cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
    sim = EventSimulator(W, H, streams=S, frames_per_step=T, config=cfg)
    f0 = [texture_frame(W, H, 0.137 * s) for s in range(S)]
    sim.reset(f0, seeds=list(range(S)))
    ost = [oracle.init_state(f0[s], c_pos=0.15, c_neg=0.15, refractory_us=100, seed=s) for s in range(S)]
    for step in range(2):
        frames = np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (step * T + f + 1)) for f in range(T)]
                           for s in range(S)])
        out = sim.step_host(frames)
        for s in range(S):
            for f in range(T):
                k = step * T + f
                ob = oracle.canonical_sort(oracle.generate(ost[s], frames[s, f], k * 1000, (k + 1) * 1000,
                                                           refractory_us=100))
                assert out[s][f].same_events(ob), (step, s, f)


def test_run_host_pipeline_matches_oracle():
    """Pipelined host stepping (EventSimulator.run_host, pinned source windows)."""
    import numpy as np

    from paper_2602_15018_b200.simulator import EventSimulator

    S, T, H, W = 2, 3, 36, 48
    cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
    sim = EventSimulator(W, H, streams=S, frames_per_step=T, config=cfg)
    f0 = [texture_frame(W, H, 0.137 * s) for s in range(S)]
    sim.reset(f0, seeds=list(range(S)))
    ost = [oracle.init_state(f0[s], c_pos=0.15, c_neg=0.15, refractory_us=100, seed=s) for s in range(S)]
    nwin = 5
    wins = [np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (w * T + f + 1)) for f in range(T)]
                      for s in range(S)]) for w in range(nwin)]
    for w in wins:
        EventSimulator.pin_host(w)
    try:
        got = list(sim.run_host(wins))
    finally:
        for w in wins:
            EventSimulator.unpin_host(w)
    assert len(got) == nwin
    for w in range(nwin):
        for s in range(S):
            for f in range(T):
                k = w * T + f
                ob = oracle.canonical_sort(oracle.generate(ost[s], wins[w][s, f], k * 1000, (k + 1) * 1000,
                                                           refractory_us=100))
                assert got[w][s][f].same_events(ob), (w, s, f)


@pytest.mark.parametrize("noise_cap,canonical", [
    (None, True), (8, True),   # 8: every noise buffer overflows -> retrying path
    (None, False)])
def test_voxel_window_signal_plus_noise_matches_oracle(noise_cap, canonical):
    """EventSimulator.voxel_window: the T frames' signal events plus per-frame
    exact noise of one window, accumulated without sorting / merging, equals
    the oracle's voxel grid of the concatenated window batch."""
    import torch

    from paper_2602_15018_b200.simulator import EventSimulator, mix64

    S, T, W, H = 2, 4, 160, 96
    cfg = ev.EventCameraConfig(c_pos=0.05, c_neg=0.05, refractory_us=0, noise_rate_hz=2000.0)
    sim = EventSimulator(W, H, streams=S, frames_per_step=T, config=cfg, canonical=canonical)
    f0 = [texture_frame(W, H, 0.3 + 0.137 * s) for s in range(S)]
    sim.reset(f0, seeds=[5 + s for s in range(S)])
    ost = [oracle.init_state(f0[s], c_pos=0.05, c_neg=0.05, seed=5 + s) for s in range(S)]
    k = 0
    for step in range(2):
        frames = np.stack([[texture_frame(W, H, 0.3 + 0.137 * s + 0.02 * (k + f + 1)) for f in range(T)]
                           for s in range(S)])
        sim.step(torch.from_numpy(frames).cuda())
        for s in range(S):
            seeds = [mix64(7 + s, 0x6E6F6973, k + f) for f in range(T)]
            parts = []
            for f in range(T):
                t_prev, t_now = (k + f) * 1000, (k + f + 1) * 1000
                parts.append(oracle.generate(ost[s], frames[s, f], t_prev, t_now))
                parts.append(oracle.noise(W, H, t_prev, t_now, cfg.noise_rate_hz, seeds[f]))
            exp = oracle.voxel(oracle.concat(parts), k * 1000, (k + T) * 1000, 5, W, H)
            got = sim.voxel_window(s, bins=5, noise_seeds=seeds, _noise_capacity=noise_cap).cpu().numpy()
            np.testing.assert_array_equal(got, exp)
            sig_only = sim.voxel_window(s, bins=5).cpu().numpy()
            exp_sig = oracle.voxel(oracle.concat(parts[0::2]), k * 1000, (k + T) * 1000, 5, W, H)
            np.testing.assert_array_equal(sig_only, exp_sig)
        k += T


def test_voxel_window_wide_window_64bit_bins():
    """(B-1) * window >= 2^30 us: the 64-bit bin arithmetic of evs_step_voxel."""
    import torch

    from paper_2602_15018_b200.simulator import EventSimulator

    T, W, H, tick = 2, 96, 64, 300_000_000
    cfg = ev.EventCameraConfig(c_pos=0.1, c_neg=0.1, refractory_us=0)
    sim = EventSimulator(W, H, streams=1, frames_per_step=T, config=cfg, tick_us=tick)
    f0 = texture_frame(W, H, 0.2)
    sim.reset([f0], seeds=[3])
    ost = oracle.init_state(f0, c_pos=0.1, c_neg=0.1, seed=3)
    frames = np.stack([[texture_frame(W, H, 0.2 + 0.03 * (f + 1)) for f in range(T)]])
    sim.step(torch.from_numpy(frames).cuda())
    parts = [oracle.generate(ost, frames[0, f], f * tick, (f + 1) * tick) for f in range(T)]
    exp = oracle.voxel(oracle.concat(parts), 0, T * tick, 5, W, H)
    np.testing.assert_array_equal(sim.voxel_window(0, bins=5).cpu().numpy(), exp)


def test_histograms_all_streams_match_oracle():
    """EventSimulator.histograms: accumulate_events_to_image of every stream in
    one launch, windows inside and across the step's frames."""
    import torch

    from paper_2602_15018_b200.simulator import EventSimulator

    S, T, W, H = 5, 3, 346, 260
    cfg = ev.EventCameraConfig(c_pos=0.2, c_neg=0.2, refractory_us=0)
    sim = EventSimulator(W, H, streams=S, frames_per_step=T, config=cfg)
    f0 = [texture_frame(W, H, 0.137 * s) for s in range(S)]
    sim.reset(f0, seeds=list(range(S)))
    ost = [oracle.init_state(f0[s], seed=s) for s in range(S)]
    frames = np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (f + 1)) for f in range(T)] for s in range(S)])
    sim.step(torch.from_numpy(frames).cuda())
    batches = [oracle.concat([oracle.generate(ost[s], frames[s, f], f * 1000, (f + 1) * 1000)
                              for f in range(T)]) for s in range(S)]
    for window, t_end in ((2000, 3000), (1500, 2200), (10, 1), (5000, 3000)):
        got = sim.histograms(window, t_end).cpu().numpy()
        for s in range(S):
            assert np.array_equal(got[s], oracle.accumulate(batches[s], window, t_end, W, H)), (window, t_end, s)
    assert np.array_equal(sim.histograms(1000).cpu().numpy()[2],
                          oracle.accumulate(batches[2], 1000, 3000, W, H))
