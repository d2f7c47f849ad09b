"""Row-band split on the GPU: several GpuBand slices of one sensor stepped by
the evs_step kernels (LocalBands: same planning as the multi-rank BandedCamera)
against the unsplit CPU oracle, including the capacity cut and invalid frames."""

import numpy as np
import pytest

import oracle
from paper_2602_15018_b200 import events as ev
from paper_2602_15018_b200.bands import GpuBand, LocalBands, band_rows
from paper_2602_15018_b200.events.parallel import AggregationStats
from paper_2602_15018_b200.synth import texture_frame

pytestmark = pytest.mark.gpu


def _setup(W, H, nb, c, sigma, refr, cap, seed=3):
    cfg = ev.EventCameraConfig(c_pos=c, c_neg=c * 1.1, sigma_c=sigma, refractory_us=refr,
                               max_events_per_frame=cap)
    f0 = texture_frame(W, H, 0.1)
    st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, f0), cfg, seed=seed)
    bands = [GpuBand(st, rows, cfg) for rows in band_rows(H, W, nb)]
    full = oracle.init_state(f0, c_pos=c, c_neg=c * 1.1, sigma_c=sigma, refractory_us=refr, seed=seed)
    return cfg, LocalBands(bands, cfg, W, H), bands, full


@pytest.mark.parametrize("W,H,nb,c,sigma,refr,cap", [
    (1280, 720, 2, 0.15, 0.0, 100, None),   # BASELINE config 2 split in two bands
    (346, 260, 3, 0.2, 0.03, 0, None),      # W % 32 != 0: 16-row band granularity
    (160, 120, 4, 0.05, 0.0, 250, None),    # multi-crossing
    (160, 120, 3, 0.05, 0.0, 0, 3000),      # capacity cut inside a middle band
])
def test_bands_match_unsplit_oracle(W, H, nb, c, sigma, refr, cap):
    cfg, cam, bands, full = _setup(W, H, nb, c, sigma, refr, cap)
    capv = cfg.capacity(W, H)
    dropped_seen = 0
    for k in range(1, 5):
        fr = texture_frame(W, H, 0.1 + 0.02 * k)
        stats = AggregationStats()
        b = cam.step(fr, (k - 1) * 1000, k * 1000, stats=stats)
        exp = oracle.canonical_sort(oracle.generate(full, fr, (k - 1) * 1000, k * 1000,
                                                    refractory_us=refr, cap=capv))
        assert b.same_events(exp), k
        assert b.dropped_count == exp.dropped_count
        assert stats.reservation_count == exp.reservation_count and stats.events_emitted == len(exp)
        dropped_seen += exp.dropped_count
        for band in bands:
            sl = slice(band.y0, band.y1)
            assert np.array_equal(band.state.d_ref_log.cpu().numpy(), full.ref_log[sl])
            assert np.array_equal(band.state.d_last_event_t.cpu().numpy(), full.last_event_t[sl])
    if cap is not None:
        assert dropped_seen > 0


def test_bands_invalid_frame_raises_first_pixel_and_keeps_state():
    W, H = 160, 120
    cfg, cam, bands, full = _setup(W, H, 3, 0.1, 0.0, 100, None)
    cam.step(texture_frame(W, H, 0.12), 0, 1000)
    before = [(b.state.d_ref_log.clone(), b.state.d_last_event_t.clone()) for b in bands]
    fr = texture_frame(W, H, 0.14)
    fr[70, 9] = np.inf    # band 1
    fr[100, 3] = -0.5     # band 2
    with pytest.raises(ValueError, match=r"\(x=9, y=70\)"):
        cam.step(fr, 1000, 2000)
    for b, (r, l) in zip(bands, before):
        assert np.array_equal(b.state.d_ref_log.cpu().numpy(), r.cpu().numpy())
        assert np.array_equal(b.state.d_last_event_t.cpu().numpy(), l.cpu().numpy())


def test_bands_device_output():
    W, H = 346, 260
    cfg, cam, bands, full = _setup(W, H, 2, 0.2, 0.0, 0, None)
    fr = texture_frame(W, H, 0.13)
    d = cam.step(fr, 0, 1000, device_output=True)
    exp = oracle.canonical_sort(oracle.generate(full, fr, 0, 1000, cap=cfg.capacity(W, H)))
    assert d.to_host().same_events(exp)
