"""Batched engine (S streams x T frames per launch), device clock + CUDA-graph
replay, against the CPU oracle frame by frame."""

import numpy as np
import pytest

import oracle
from paper_2602_15018_b200 import _lib
from paper_2602_15018_b200.runtime import StepEngine, StepShape
from paper_2602_15018_b200.synth import texture_frame

pytestmark = pytest.mark.gpu


def _setup(S, T, H, W, cfg, seeds, sigma=0.0, refr=0, order=1, nframes=None):
    import torch

    nframes = nframes or T
    frames = np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (k + 1)) for k in range(nframes)]
                       for s in range(S)])
    ost = [oracle.init_state(texture_frame(W, H, 0.137 * s), c_pos=cfg[0], c_neg=cfg[1], sigma_c=sigma,
                             refractory_us=refr, seed=seeds[s]) for s in range(S)]
    dev = torch.device("cuda")
    ref = torch.from_numpy(np.stack([o.ref_log for o in ost])).to(dev)
    last = torch.from_numpy(np.stack([o.last_event_t for o in ost])).to(dev)
    thp = torch.from_numpy(np.stack([o.thresholds_pos for o in ost])).to(dev)
    thn = torch.from_numpy(np.stack([o.thresholds_neg for o in ost])).to(dev)
    uniform = (float(cfg[0]), float(cfg[1])) if sigma == 0 else None
    shape = StepShape(S, T, H, W, 8 * H * W, order, 1000, 0.01, refr, uniform)
    eng = StepEngine(shape, dev)
    return frames, ost, ref, last, thp, thn, eng


def _check_segment(eng, seg, ob, order):
    counts, dropped, res, bad = eng.fetch_info()
    assert bad == _lib.NO_BAD
    n = int(counts[seg])
    assert n == len(ob), (seg, n, len(ob))
    t = eng.ev_t[seg, :n].cpu().numpy()
    x = eng.ev_x[seg, :n].cpu().numpy().view(np.uint16)
    y = eng.ev_y[seg, :n].cpu().numpy().view(np.uint16)
    p = eng.ev_p[seg, :n].cpu().numpy()
    exp = oracle.canonical_sort(ob) if order == 1 else ob
    assert np.array_equal(t, exp.t.astype(np.int64))
    assert np.array_equal(x, exp.x) and np.array_equal(y, exp.y) and np.array_equal(p, exp.polarity)
    assert int(res[seg]) == ob.reservation_count
    assert int(dropped[seg]) == ob.dropped_count


@pytest.mark.parametrize("S,T,H,W,sigma,refr,order", [
    (1, 4, 90, 160, 0.0, 100, 1),
    (3, 5, 48, 64, 0.03, 0, 1),
    (2, 3, 37, 53, 0.03, 250, 1),     # ragged: P % 4 != 0, scalar path
    (2, 4, 48, 64, 0.0, 100, 0),      # pixel-major (serial) order
])
def test_batched_matches_oracle(S, T, H, W, sigma, refr, order):
    import torch

    cfg = (0.15, 0.15)
    frames, ost, ref, last, thp, thn, eng = _setup(S, T, H, W, cfg, list(range(S)), sigma, refr, order)
    dframes = torch.from_numpy(frames).cuda()
    eng.launch(dframes, ref, last, thp, thn, t0=0, tick=1000)
    torch.cuda.synchronize()
    for s in range(S):
        for f in range(T):
            ob = oracle.generate(ost[s], frames[s, f], f * 1000, (f + 1) * 1000, refractory_us=refr)
            _check_segment(eng, s * T + f, ob, order)
        assert np.array_equal(ref[s].cpu().numpy(), ost[s].ref_log)
        assert np.array_equal(last[s].cpu().numpy(), ost[s].last_event_t)


def test_t_bounds_irregular_ticks():
    import torch

    S, T, H, W = 2, 3, 32, 48
    frames, ost, ref, last, thp, thn, eng = _setup(S, T, H, W, (0.2, 0.2), [0, 1], 0.0, 100, 1)
    tb = np.array([[0, 700, 1900, 2500], [100, 1100, 1300, 4000]], np.int64)
    shape = StepShape(S, T, H, W, 8 * H * W, 1, 4096, 0.01, 100, (0.2, 0.2))
    eng = StepEngine(shape, ref.device)
    eng.launch(torch.from_numpy(frames).cuda(), ref, last, t_bounds=torch.from_numpy(tb).cuda())
    torch.cuda.synchronize()
    for s in range(S):
        for f in range(T):
            ob = oracle.generate(ost[s], frames[s, f], int(tb[s, f]), int(tb[s, f + 1]), refractory_us=100)
            _check_segment(eng, s * T + f, ob, 1)


def test_graph_replay_matches_oracle():
    """Device clock + CUDA graph: 3 replays of a 4-step graph == 12 oracle frames."""
    import torch

    H, W = 64, 96
    nfr = 4
    frames, ost, ref, last, thp, thn, eng = _setup(1, 1, H, W, (0.15, 0.15), [7], 0.0, 100, 1, nframes=nfr)
    dfr = torch.from_numpy(frames[0]).cuda()
    windows = [dfr[i:i + 1] for i in range(nfr)]
    eng.launch(windows[0], ref, last, t0=0, tick=1000)  # eager step 0
    torch.cuda.synchronize()
    ob = oracle.generate(ost[0], frames[0, 0], 0, 1000, refractory_us=100)
    _check_segment(eng, 0, ob, 1)
    order = [1, 2, 3, 0]
    eng.capture([windows[i] for i in order], ref, last, tick=1000, t0=1000)
    k = 1
    for _rep in range(3):
        eng.replay()
        torch.cuda.synchronize()
        for i in order:
            ob = oracle.generate(ost[0], frames[0, i], k * 1000, (k + 1) * 1000, refractory_us=100)
            k += 1
        # the engine's output holds the last step of the replay
        _check_segment(eng, 0, ob, 1)
        assert np.array_equal(ref[0].cpu().numpy(), ost[0].ref_log)
        assert np.array_equal(last[0].cpu().numpy(), ost[0].last_event_t)
    # eager launches continue the same sequence after graph replays
    eng.launch(windows[1], ref, last, t0=k * 1000, tick=1000)
    torch.cuda.synchronize()
    ob = oracle.generate(ost[0], frames[0, 1], k * 1000, (k + 1) * 1000, refractory_us=100)
    _check_segment(eng, 0, ob, 1)


@pytest.mark.parametrize("T", [2, 5])  # prologue validation (T < 4) / fused into K1 (T >= 4)
def test_invalid_frame_leaves_state_untouched(T):
    import torch

    H, W = 16, 24
    frames, ost, ref, last, thp, thn, eng = _setup(2, T, H, W, (0.2, 0.2), [0, 1])
    frames[1, 1, 3, 5] = np.nan
    frames[1, 1, 7, 2] = 2.0
    ref0, last0 = ref.clone(), last.clone()
    eng.launch(torch.from_numpy(frames).cuda(), ref, last, t0=0, tick=1000)
    counts, dropped, res, bad = eng.fetch_info()
    assert bad == (1 * T + 1) * H * W + 3 * W + 5
    assert torch.equal(ref, ref0) and torch.equal(last, last0)
    assert int(counts.sum()) == 0


def test_infinite_intensity_rejected_fast_and_state_kept():
    """+inf / huge values: the call is rejected (first bad pixel) without
    running the crossing loops on them (an inf once meant ~2^31 crossings)."""
    import time

    import torch

    H, W = 40, 160
    for T in (1, 5):
        frames, ost, ref, last, thp, thn, eng = _setup(1, T, H, W, (0.1, 0.1), [0])
        frames[0, 0, 20, 9] = np.inf
        frames[0, T - 1, 3, 4] = 1e30
        ref0, last0 = ref.clone(), last.clone()
        t0 = time.time()
        eng.launch(torch.from_numpy(frames).cuda(), ref, last, t0=0, tick=1000)
        counts, dropped, res, bad = eng.fetch_info()
        assert time.time() - t0 < 5.0
        assert bad == (3 * W + 4 if T == 1 else 20 * W + 9)
        assert torch.equal(ref, ref0) and torch.equal(last, last0)


def test_corrupt_reference_level_fails_loudly():
    import torch

    from paper_2602_15018_b200._lib import NativeError

    H, W = 16, 64
    frames, ost, ref, last, thp, thn, eng = _setup(1, 1, H, W, (0.1, 0.1), [0])
    ref[0, 5, 7] = -1e30  # |diff| / th ~ 1e31 crossings
    eng.launch(torch.from_numpy(frames).cuda(), ref, last, t0=0, tick=1000)
    with pytest.raises(NativeError, match="2\\*\\*20"):
        eng.fetch_info()
