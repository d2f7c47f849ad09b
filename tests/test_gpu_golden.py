"""CUDA path (through the C ABI) against the reference's golden vectors."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GEN_CASES = ["texture_davis", "texture_refr_canon", "walk_sigma", "walk_refr", "walk_cap", "walk_multi"]


@pytest.mark.parametrize("case", GEN_CASES)
@pytest.mark.parametrize("api", ["serial", "parallel"])
def test_generate_matches_reference_golden(case, api):
    from paper_2602_15018_b200 import events as ev

    g = dict(np.load(os.path.join(GOLD, f"gen_{case}.npz")))
    c_pos, c_neg, sigma, refr, log_eps, cap = g["cfg"]
    cfg = ev.EventCameraConfig(c_pos=c_pos, c_neg=c_neg, sigma_c=sigma, refractory_us=int(refr),
                               log_eps=log_eps, max_events_per_frame=int(cap))
    h, w = g["frames"].shape[1:]
    st = ev.PixelStateGrid(w, h, g["ref0"], g["last0"], g["thp"], g["thn"])
    off = 0
    for k in range(1, len(g["frames"])):
        fr = ev.IntensityFrame(width=w, height=h, t=int(g["times"][k]), values=g["frames"][k])
        stats = ev.AggregationStats()
        if api == "serial":
            b = ev.generate_events_serial(st, fr, int(g["times"][k - 1]), int(g["times"][k]), cfg)
        else:
            b = ev.generate_events_parallel(st, fr, int(g["times"][k - 1]), int(g["times"][k]), cfg,
                                            workers=4, stats=stats)
        n = int(g["ev_n"][k - 1])
        exp = ev.EventBatch(g["ev_t"][off:off + n].astype(np.uint64), g["ev_x"][off:off + n],
                            g["ev_y"][off:off + n], g["ev_p"][off:off + n])
        off += n
        if api == "parallel" or not bool(g["serial"]):
            # parallel output is canonical; compare canonical forms
            exp = ev.canonical_sort(exp)
            got = b if api == "parallel" else ev.canonical_sort(b)
        else:
            got = b
        assert got.same_events(exp), (case, api, k, len(got), n)
        assert b.dropped_count == int(g["dropped"][k - 1])
        if api == "parallel" and int(g["res"][k - 1]) >= 0:
            assert stats.reservation_count == int(g["res"][k - 1])
        assert np.array_equal(st.ref_log, g["refs"][k - 1])
        assert np.array_equal(st.last_event_t, g["lasts"][k - 1])


def test_canonical_sort_golden():
    from paper_2602_15018_b200 import events as ev

    g = dict(np.load(os.path.join(GOLD, "batch_ops.npz")))
    b = ev.EventBatch(g["t"].astype(np.uint64), g["x"], g["y"], g["p"], dropped_count=4)
    cs = ev.canonical_sort(b)
    assert cs.dropped_count == 4
    assert np.array_equal(cs.t.astype(np.int64), g["cs_t"]) and np.array_equal(cs.x, g["cs_x"])
    assert np.array_equal(cs.y, g["cs_y"]) and np.array_equal(cs.polarity, g["cs_p"])
