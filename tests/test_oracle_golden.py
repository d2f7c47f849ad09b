"""The CPU oracle (oracle/) against golden vectors produced by the reference itself.

CPU-only: pins the oracle before it is trusted as the checker of the CUDA path.
"""

import os
import sys

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GEN_CASES = ["texture_davis", "texture_refr_canon", "walk_sigma", "walk_refr", "walk_cap", "walk_multi"]


def load(name):
    return dict(np.load(os.path.join(GOLD, name), allow_pickle=False))


@pytest.mark.parametrize("case", GEN_CASES)
def test_oracle_generate_matches_reference(oracle_mod, case):
    g = load(f"gen_{case}.npz")
    c_pos, c_neg, sigma, refr, log_eps, cap = g["cfg"]
    st = oracle_mod.OState(g["frames"].shape[2], g["frames"].shape[1], g["ref0"].copy(),
                           g["last0"].copy(), g["thp"], g["thn"])
    off = 0
    for k in range(1, len(g["frames"])):
        b = oracle_mod.generate(st, g["frames"][k], int(g["times"][k - 1]), int(g["times"][k]),
                                log_eps=log_eps, refractory_us=int(refr), cap=int(cap))
        n = int(g["ev_n"][k - 1])
        exp = oracle_mod.OBatch(g["ev_t"][off:off + n].astype(np.uint64), g["ev_x"][off:off + n],
                                g["ev_y"][off:off + n], g["ev_p"][off:off + n])
        off += n
        got = b if bool(g["serial"]) else oracle_mod.canonical_sort(b)
        assert got.same_events(exp), (case, k)
        assert b.dropped_count == int(g["dropped"][k - 1])
        if int(g["res"][k - 1]) >= 0:
            assert b.reservation_count == int(g["res"][k - 1])
        assert np.array_equal(st.ref_log, g["refs"][k - 1])
        assert np.array_equal(st.last_event_t, g["lasts"][k - 1])


def test_oracle_noise_matches_reference(oracle_mod):
    g = load("noise.npz")
    i = 0
    while f"case{i}" in g:
        w, h, t0, t1, seed = [int(v) for v in g[f"case{i}"]]
        b = oracle_mod.noise(w, h, t0, t1, float(g[f"rate{i}"][0]), seed)
        assert np.array_equal(b.t.astype(np.int64), g[f"t{i}"]), i
        assert np.array_equal(b.x, g[f"x{i}"]) and np.array_equal(b.y, g[f"y{i}"])
        assert np.array_equal(b.polarity, g[f"p{i}"])
        i += 1
    assert i >= 5


def test_oracle_pcg64_seeding(oracle_mod):
    g = np.load(os.path.join(GOLD, "pcg64.npz"))
    for s, st in zip(g["seeds"], g["states"]):
        assert np.array_equal(oracle_mod.pcg64_state(int(s)), st), s
    assert np.array_equal(oracle_mod.pcg64_draws(99, 64), g["raw99"])


def test_oracle_batch_ops(oracle_mod):
    g = load("batch_ops.npz")
    b = oracle_mod.OBatch(g["t"].astype(np.uint64), g["x"], g["y"], g["p"], 4)
    cs = oracle_mod.canonical_sort(b)
    assert np.array_equal(cs.t.astype(np.int64), g["cs_t"]) and np.array_equal(cs.x, g["cs_x"])
    assert np.array_equal(cs.y, g["cs_y"]) and np.array_equal(cs.polarity, g["cs_p"])
    assert np.array_equal(oracle_mod.accumulate(b, 1500, 2500, 40, 30), g["acc"])
    lb = oracle_mod.limit_bandwidth(cs, 2.0e6, 100)
    assert np.array_equal(lb.t.astype(np.int64), g["lb_t"])
    assert lb.dropped_count == int(g["lb_dropped"][0])


def test_oracle_multithreaded_equals_serial(oracle_mod):
    g = load("gen_walk_multi.npz")
    c_pos, c_neg, sigma, refr, log_eps, cap = g["cfg"]
    mk = lambda: oracle_mod.OState(40, 30, g["ref0"].copy(), g["last0"].copy(), g["thp"], g["thn"])
    a, b = mk(), mk()
    for k in range(1, len(g["frames"])):
        x = oracle_mod.generate(a, g["frames"][k], int(g["times"][k - 1]), int(g["times"][k]),
                                log_eps=log_eps, refractory_us=int(refr), cap=int(cap))
        y = oracle_mod.generate(b, g["frames"][k], int(g["times"][k - 1]), int(g["times"][k]),
                                log_eps=log_eps, refractory_us=int(refr), cap=int(cap), nthreads=3)
        assert x.same_events(y) and x.reservation_count == y.reservation_count
        assert np.array_equal(a.ref_log, b.ref_log)


def test_oracle_voxel_definition(oracle_mod):
    # two events in a 1-pixel window [0, 100) with 5 bins: exact bilinear weights
    b = oracle_mod.OBatch(np.array([0, 50], np.uint64), np.zeros(2, np.uint16), np.zeros(2, np.uint16),
                          np.array([1, -1], np.int8))
    v = oracle_mod.voxel(b, 0, 100, 5, 1, 1)[:, 0, 0]
    # t=0 -> tau=0 -> bin0 weight 1 ; t=50 -> tau=2 (bins of 25us) -> bin2 weight -1
    np.testing.assert_array_equal(v, np.array([1.0, 0.0, -1.0, 0.0, 0.0], np.float32))


def test_bench_fixture_first_frames_from_oracle(oracle_mod):
    """tests/golden/bench_hd_t50.json (bench.py's self-check fixture) is the
    oracle's output: its first frames recomputed here (CPU)."""
    import json
    import os

    from paper_2602_15018_b200.synth import texture_frame

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    from make_bench_golden import batch_sha1

    with open(os.path.join(here, "bench_hd_t50.json")) as f:
        fx = json.load(f)
    W, H = 1280, 720
    oracle = oracle_mod
    st = oracle.init_state(texture_frame(W, H, 0.0), c_pos=0.15, c_neg=0.15, refractory_us=100, seed=0)
    for j in range(4):
        b = oracle.canonical_sort(oracle.generate(st, texture_frame(W, H, 0.02 * j), j * 1000, (j + 1) * 1000,
                                                  refractory_us=100))
        assert fx["frames"][j] == {"count": len(b), "dropped": b.dropped_count,
                                   "reservations": b.reservation_count,
                                   "sha1": batch_sha1(b.t, b.x, b.y, b.polarity)}, j


def test_oracle_canonical_sort_general(oracle_mod):
    """The oracle's canonical_sort (uint64 t, int8 polarity) vs the reference's
    lexsort on a batch outside the simulator's range (sort_general.npz)."""
    g = load("sort_general.npz")
    b = oracle_mod.canonical_sort(oracle_mod.OBatch(g["t"].view(np.uint64), g["x"], g["y"], g["p"]))
    assert np.array_equal(b.t.view(np.int64), g["cs_t"]) and np.array_equal(b.x, g["cs_x"])
    assert np.array_equal(b.y, g["cs_y"]) and np.array_equal(b.polarity, g["cs_p"])
