"""Fast canonical path (csrc/fast_path.cu) against the CPU oracle and against the
tile-order path (the default, exact-f64 lane math), including its rare paths: tile
lists that overflow shared memory, the capacity cut, irregular ticks, and
random inputs that stress the certified f32 lane math."""

import os

import numpy as np
import pytest

import oracle
from paper_2602_15018_b200 import _lib
from paper_2602_15018_b200.runtime import StepEngine, StepShape
from paper_2602_15018_b200.synth import texture_frame

pytestmark = pytest.mark.gpu


def _run(frames, ref0, last0, thp, thn, refr, cap, uniform, legacy=False, t_bounds=None, tick=1000,
         max_dt=1024):
    """One StepEngine launch over frames [S][T][H][W]; returns outputs + new state."""
    import torch

    S, T, H, W = frames.shape
    dev = torch.device("cuda")
    old = os.environ.get("EVS_PATH")
    if legacy:
        os.environ.pop("EVS_PATH", None)
    else:
        os.environ["EVS_PATH"] = "bucket"

    try:
        eng = StepEngine(StepShape(S, T, H, W, cap, 1, max_dt, 0.01, refr, uniform), dev)
        ref = torch.from_numpy(ref0.copy()).to(dev)
        last = torch.from_numpy(last0.copy()).to(dev)
        tp = torch.from_numpy(thp).to(dev) if uniform is None else None
        tn = torch.from_numpy(thn).to(dev) if uniform is None else None
        tbd = torch.from_numpy(t_bounds).to(dev) if t_bounds is not None else None
        eng.launch(torch.from_numpy(frames).to(dev), ref, last, tp, tn, t_bounds=tbd, t0=0, tick=tick)
        counts, dropped, res, bad = eng.fetch_info()
    finally:
        if old is None:
            os.environ.pop("EVS_PATH", None)
        else:
            os.environ["EVS_PATH"] = old
    assert bad == _lib.NO_BAD
    segs = []
    for g in range(S * T):
        n = int(counts[g])
        segs.append((eng.ev_t[g, :n].cpu().numpy(), eng.ev_x[g, :n].cpu().numpy().view(np.uint16),
                     eng.ev_y[g, :n].cpu().numpy().view(np.uint16), eng.ev_p[g, :n].cpu().numpy(),
                     int(dropped[g]), int(res[g])))
    return segs, ref.cpu().numpy(), last.cpu().numpy()


def _oracle_segments(frames, ref0, last0, thp, thn, refr, cap, t_bounds=None, tick=1000):
    S, T, H, W = frames.shape
    out = []
    refs, lasts = [], []
    for s in range(S):
        st = oracle.OState(W, H, ref0[s].copy(), last0[s].copy(), thp[s].copy(), thn[s].copy())
        for f in range(T):
            t0, t1 = ((int(t_bounds[s, f]), int(t_bounds[s, f + 1])) if t_bounds is not None
                      else (f * tick, (f + 1) * tick))
            ob = oracle.canonical_sort(oracle.generate(st, frames[s, f], t0, t1, refractory_us=refr, cap=cap))
            out.append(ob)
        refs.append(st.ref_log)
        lasts.append(st.last_event_t)
    return out, np.stack(refs), np.stack(lasts)


def _same(segs, exp):
    for g, (got, ob) in enumerate(zip(segs, exp)):
        t, x, y, p, dropped, res = got
        assert len(t) == len(ob), (g, len(t), len(ob))
        assert np.array_equal(t, ob.t.astype(np.int64)), g
        assert np.array_equal(x, ob.x) and np.array_equal(y, ob.y), g
        assert np.array_equal(p, ob.polarity), g
        assert dropped == ob.dropped_count, (g, dropped, ob.dropped_count)
        assert res == ob.reservation_count, (g, res, ob.reservation_count)


def _texture_case(S, T, H, W, c, refr, sigma=0.0):
    frames = np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (k + 1)) for k in range(T)] for s in range(S)])
    sts = [oracle.init_state(texture_frame(W, H, 0.137 * s), c_pos=c, c_neg=c, sigma_c=sigma,
                             refractory_us=refr, seed=s) for s in range(S)]
    ref0 = np.stack([o.ref_log for o in sts])
    last0 = np.stack([o.last_event_t for o in sts])
    thp = np.stack([o.thresholds_pos for o in sts])
    thn = np.stack([o.thresholds_neg for o in sts])
    return frames, ref0, last0, thp, thn


PATHS = pytest.mark.parametrize("bucket", [True, False], ids=["bucket", "tile"])


@PATHS
@pytest.mark.parametrize("S,T,H,W,c,refr,sigma", [
    (1, 3, 720, 1280, 0.15, 100, 0.0),   # BASELINE config 2 shape
    (1, 1, 720, 1280, 0.15, 100, 0.0),   # one frame per call (4-tile groups, prologue validation)
    (2, 4, 260, 346, 0.2, 0, 0.0),       # DAVIS
    (2, 3, 120, 160, 0.05, 0, 0.03),     # multi-crossing, non-uniform thresholds
    (1, 2, 33, 37, 0.1, 300, 0.0),       # ragged tiles, scalar loads
])
def test_fast_matches_oracle(S, T, H, W, c, refr, sigma, bucket):
    frames, ref0, last0, thp, thn = _texture_case(S, T, H, W, c, refr, sigma)
    cap = 8 * H * W
    uniform = (c, c) if sigma == 0 else None
    segs, ref, last = _run(frames, ref0, last0, thp, thn, refr, cap, uniform, legacy=not bucket)
    exp, oref, olast = _oracle_segments(frames, ref0, last0, thp, thn, refr, cap)
    _same(segs, exp)
    assert np.array_equal(ref, oref) and np.array_equal(last, olast)


def test_random_inputs_fast_equals_exact_path():
    """Uniform random frames / levels: many pixels near floor boundaries; the
    certified f32 math must agree bit for bit with the exact f64 path."""
    rng = np.random.default_rng(5)
    S, T, H, W = 2, 3, 256, 384
    # a random walk in log intensity: diverse fractional parts of |diff|/th and
    # of the crossing times, a few crossings per pixel
    L = np.log(rng.random((S, H, W)) * 0.9 + 0.05)
    ref0 = (L + rng.normal(0.0, 0.2, (S, H, W))).astype(np.float32)
    frames = np.empty((S, T, H, W), np.float32)
    for f in range(T):
        L = np.clip(L + rng.normal(0.0, 0.25, (S, H, W)), np.log(0.02), 0.0)
        frames[:, f] = np.clip(np.exp(L) - 0.01, 0.0, 1.0)
    last0 = rng.integers(-3000, 500, (S, H, W)).astype(np.int64)
    thp = np.maximum(rng.normal(0.1, 0.05, (S, H, W)), 0.01).astype(np.float32)
    thn = np.maximum(rng.normal(0.12, 0.05, (S, H, W)), 0.01).astype(np.float32)
    cap = 8 * H * W
    for refr in (0, 150):
        a = _run(frames, ref0, last0, thp, thn, refr, cap, None)
        b = _run(frames, ref0, last0, thp, thn, refr, cap, None, legacy=True)
        for sa, sb in zip(a[0], b[0]):
            for u, v in zip(sa, sb):
                assert np.array_equal(np.asarray(u), np.asarray(v))
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
        exp, oref, olast = _oracle_segments(frames, ref0, last0, thp, thn, refr, cap)
        _same(a[0], exp)
        assert np.array_equal(a[1], oref) and np.array_equal(a[2], olast)


def test_tile_order_overflow_area_within_capacity():
    """~6 crossings per pixel (under the capacity): every tile-order region
    overflows (> 4096 events per 1024-pixel tile) into the overflow area, whose
    keys K2 and k_group_hist then read."""
    rng = np.random.default_rng(4)
    S, T, H, W = 1, 2, 64, 96
    L0 = rng.uniform(-3.0, -2.0, (H, W))
    ref0 = L0.astype(np.float32)[None]
    f1 = oracle.frame_from_log(L0 + rng.uniform(0.055, 0.075, (H, W)))
    f2 = oracle.frame_from_log(L0 + rng.uniform(0.0, 0.02, (H, W)))
    frames = np.stack([[f1, f2]]).astype(np.float32)
    last0 = np.full((1, H, W), -100, np.int64)
    thp = np.full((1, H, W), 0.01, np.float32)
    thn = np.full((1, H, W), 0.011, np.float32)
    cap = 8 * H * W
    for refr in (0, 3):
        segs, ref, last = _run(frames, ref0, last0, thp, thn, refr, cap, (0.01, 0.011), legacy=True)
        exp, oref, olast = _oracle_segments(frames, ref0, last0, thp, thn, refr, cap)
        assert len(exp[0]) > 5 * H * W  # > 4096 per 1024-pixel tile
        _same(segs, exp)
        assert np.array_equal(ref, oref) and np.array_equal(last, olast)


@PATHS
def test_overflow_tiles_sorted_by_fixup(bucket):
    """> 3 crossings per pixel across whole tiles: the bucket path's tile lists
    overflow shared memory (overflow area + fixup sort).  The first frame lies
    far above its capacity, which the tile-order path reports instead
    (its overflow area holds at most the capacity + a few tiles)."""
    if not bucket:
        pytest.skip("tile-order path: see test_tile_order_overflow_area_within_capacity")
    rng = np.random.default_rng(2)
    S, T, H, W = 1, 2, 64, 96
    L0 = rng.uniform(-4.0, -3.0, (H, W))
    ref0 = L0.astype(np.float32)[None]
    f1 = oracle.frame_from_log(L0 + rng.uniform(2.0, 3.5, (H, W)))
    f2 = oracle.frame_from_log(L0 + rng.uniform(0.0, 0.8, (H, W)))
    frames = np.stack([[f1, f2]]).astype(np.float32)
    last0 = np.full((1, H, W), -100, np.int64)
    thp = np.full((1, H, W), 0.01, np.float32)
    thn = np.full((1, H, W), 0.011, np.float32)
    cap = 8 * H * W
    for refr in (0, 20):
        segs, ref, last = _run(frames, ref0, last0, thp, thn, refr, cap, (0.01, 0.011), legacy=not bucket)
        exp, oref, olast = _oracle_segments(frames, ref0, last0, thp, thn, refr, cap)
        assert max(len(e) for e in exp) > 3 * H * W  # really overflowed
        _same(segs, exp)
        assert np.array_equal(ref, oref) and np.array_equal(last, olast)


@PATHS
@pytest.mark.parametrize("cap", [1, 777, 5000, 20000])
def test_capacity_cut(cap, bucket):
    frames, ref0, last0, thp, thn = _texture_case(2, 2, 96, 128, 0.05, 0)
    segs, ref, last = _run(frames, ref0, last0, thp, thn, 0, cap, (0.05, 0.05), legacy=not bucket)
    exp, oref, olast = _oracle_segments(frames, ref0, last0, thp, thn, 0, cap)
    _same(segs, exp)
    assert np.array_equal(ref, oref) and np.array_equal(last, olast)


@PATHS
def test_irregular_ticks_and_wide_dt(bucket):
    frames, ref0, last0, thp, thn = _texture_case(2, 3, 48, 80, 0.1, 200)
    tb = np.array([[0, 700, 2600, 2601], [50, 1100, 1400, 3400]], np.int64)
    segs, ref, last = _run(frames, ref0, last0, thp, thn, 200, 8 * 48 * 80, (0.1, 0.1), t_bounds=tb,
                           max_dt=2048, legacy=not bucket)
    exp, oref, olast = _oracle_segments(frames, ref0, last0, thp, thn, 200, 8 * 48 * 80, t_bounds=tb)
    _same(segs, exp)
    assert np.array_equal(ref, oref) and np.array_equal(last, olast)


@PATHS
def test_uniform_brightness_step_single_bucket(bucket):
    """Every pixel crosses at the same instant: one t_rel bucket holds all
    events (K2 multi-chunk path, K1 single-bucket ranking)."""
    H, W = 300, 400
    ref0 = np.full((1, H, W), np.log(0.2 + 0.01), np.float32)
    frames = np.full((1, 2, H, W), 0.9, np.float32)
    frames[0, 1] = 0.95
    last0 = np.full((1, H, W), -1000, np.int64)
    thp = np.full((1, H, W), 0.2, np.float32)
    thn = thp.copy()
    cap = 8 * H * W
    segs, ref, last = _run(frames, ref0, last0, thp, thn, 0, cap, (0.2, 0.2), legacy=not bucket)
    exp, oref, olast = _oracle_segments(frames, ref0, last0, thp, thn, 0, cap)
    assert len(exp[0]) > 8192
    _same(segs, exp)
    assert np.array_equal(ref, oref) and np.array_equal(last, olast)
