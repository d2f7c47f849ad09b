"""evs_pack_segments (the gather payload of BASELINE config 5) and
evs_merge_runs (the row-band merge) against the host-side definitions."""

import numpy as np
import pytest

import oracle
from paper_2602_15018_b200 import events as ev
from paper_2602_15018_b200.synth import texture_frame

pytestmark = pytest.mark.gpu


def test_pack_segments_matches_definition():
    import torch

    from paper_2602_15018_b200.distributed import KEY64_LAYOUT, key32_layout, pack_keys, pack_segments, unpack_keys
    from paper_2602_15018_b200.simulator import EventSimulator

    W, H, S, T = 346, 260, 6, 4
    sim = EventSimulator(W, H, streams=S, frames_per_step=T, config=ev.EventCameraConfig())
    sim.reset([texture_frame(W, H, 0.137 * s) for s in range(S)])
    frames = np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (f + 1)) for f in range(T)] for s in range(S)])
    sim.step(torch.from_numpy(frames).cuda())
    r = sim.result()
    e = sim.engine
    rows = (e.ev_t, e.ev_x, e.ev_y, e.ev_p)
    counts = r.counts.ravel()
    for lay, kb in ((key32_layout(W, H, T * 1000), 4), (KEY64_LAYOUT, 8)):
        keys, offs = pack_segments(e.info[0], rows, 0, lay, kb, y_offset=0)
        offs = offs.cpu().numpy()
        assert np.array_equal(offs, np.concatenate([[0], np.cumsum(counts)]))
        for g in range(S * T):
            n = int(counts[g])
            seg = sim.segment(g // T, g % T)
            exp = pack_keys(seg.t, seg.x.to(torch.int64) & 0xFFFF, seg.y.to(torch.int64) & 0xFFFF, seg.polarity, 0,
                            lay)
            got = keys[offs[g]:offs[g] + n]
            assert torch.equal(got, exp), (kb, g)
            # key order within a segment is the canonical order (sorted, stable)
            assert bool((got[1:] >= got[:-1]).all())
            t, x, y, p = unpack_keys(got, 0, lay)
            assert torch.equal(t, seg.t) and torch.equal(p, seg.polarity)


def test_merge_runs_stable_kway():
    import torch

    from paper_2602_15018_b200.bands import merge_keys

    rng = np.random.default_rng(0)
    runs = [np.sort(rng.integers(0, 5000, n)) for n in (0, 1, 777, 20000, 3, 65000)]
    keys = torch.from_numpy(np.concatenate(runs).astype(np.int64)).cuda()
    got = merge_keys(keys, [len(r) for r in runs]).cpu().numpy()
    exp = np.sort(np.concatenate(runs), kind="stable")
    assert np.array_equal(got, exp)
