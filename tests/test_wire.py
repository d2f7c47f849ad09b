"""Events wire encoding against the reference's golden
corpus (tests/golden/events_wire.json, extracted by make_wire_golden.py from
/root/reference/pkg/golden/corpus.json) -- host path on CPU, device path on GPU."""

import json
import os

import numpy as np
import pytest

from paper_2602_15018_b200 import wire

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "events_wire.json")))


def _values(m):
    v = m["values"]
    return {
        "step_id": int(v["step_id"]), "t_us": int(v["t_us"]), "dropped": int(v["dropped"]),
        "t": np.array([int(x) for x in v["t"]["data"]], np.uint64),
        "x": np.array(v["x"]["data"], np.int64), "y": np.array(v["y"]["data"], np.int64),
        "polarity": np.array(v["polarity"]["data"], np.int64),
    }


def test_schema_hash_matches_corpus():
    assert wire.EVENTS_SCHEMA_HASH == int(GOLD["hash"], 16)


@pytest.mark.parametrize("i", range(3))
def test_host_frame_matches_golden(i):
    m = GOLD["messages"][i]
    v = _values(m)
    buf = wire.encode_events_frame(m["topic"], int(m["publish_time_ns"]), v["step_id"], v["t_us"], v)
    assert bytes(buf) == bytes.fromhex(m["frame_hex"])
    head = 1 + len(m["topic"].encode()) + 32
    assert bytes(buf[head:]) == bytes.fromhex(m["payload_hex"])
    assert len(buf) - head == wire.events_payload_size([len(v[k]) for k in ("t", "x", "y", "polarity")])


@pytest.mark.gpu
def test_device_batch_frame_matches_host_encoding():
    """A generated device batch encodes to the same bytes as its host copy."""
    from paper_2602_15018_b200 import events as ev
    from paper_2602_15018_b200.synth import texture_frame

    W, H = 96, 64
    cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15, refractory_us=100)
    st = ev.init_pixel_states(ev.IntensityFrame(W, H, 0, texture_frame(W, H, 0.0)), cfg, seed=1)
    db = ev.generate_events_parallel(st, ev.IntensityFrame(W, H, 1000, texture_frame(W, H, 0.02)), 0, 1000, cfg,
                                     device_output=True)
    hb = db.to_host() if hasattr(db, "to_host") else None
    assert len(db) > 0
    dev = wire.encode_events_frame("/sim/events", 123456789, 7, 1000, db)
    host_vals = {"t": db.t.cpu().numpy().view(np.uint64), "x": db.x.cpu().numpy().view(np.uint16),
                 "y": db.y.cpu().numpy().view(np.uint16), "polarity": db.polarity.cpu().numpy(),
                 "dropped": db.dropped_count}
    ref = wire.encode_events_frame("/sim/events", 123456789, 7, 1000, host_vals)
    assert bytes(dev) == bytes(ref)
    del hb
