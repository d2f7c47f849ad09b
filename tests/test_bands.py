"""Row-band split of one sensor (paper_2602_15018_b200/bands.py) on CPU: the
band partition, the frame planning, and the BandedCamera protocol over gloo
with 2 ranks, each band stepped by the CPU oracle (test stand-in for GpuBand),
against the unsplit oracle (generate_events_serial + canonical_sort)."""

import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2602_15018_b200.bands import (NO_BAD, BandedCamera, BandResult, TorchComm, band_rows,
                                         plan_frame)
from paper_2602_15018_b200.distributed import KEY64_LAYOUT, pack_keys
from paper_2602_15018_b200.events.parallel import AggregationStats
from paper_2602_15018_b200.events.types import EventCameraConfig


class OracleBand:
    """Rows [y0, y1) stepped by the CPU oracle (same interface as GpuBand)."""

    def __init__(self, full: oracle.OState, rows, config: EventCameraConfig):
        self.y0, self.y1 = rows
        self.width, self.height, self.sensor_height = full.width, self.y1 - self.y0, full.height
        sl = slice(self.y0, self.y1)
        self.st = oracle.OState(full.width, self.height, full.ref_log[sl].copy(), full.last_event_t[sl].copy(),
                                full.thresholds_pos[sl].copy(), full.thresholds_neg[sl].copy())
        self.config = config
        self.cap = int(config.capacity(full.width, full.height))
        self._saved = None

    def band_frame(self, frame):
        f = np.asarray(frame, np.float32)
        return f[self.y0:self.y1] if f.shape[0] == self.sensor_height else f

    def save(self):
        self._saved = (self.st.ref_log.copy(), self.st.last_event_t.copy())

    def restore(self):
        self.st.ref_log[...] = self._saved[0]
        self.st.last_event_t[...] = self._saved[1]

    def run(self, fb, t_prev, t_now, keep=None):
        empty = torch.empty(0, dtype=torch.int64)
        bad = ~np.isfinite(fb) | (fb < 0) | (fb > 1)
        if bad.any():
            flat = int(np.flatnonzero(bad.ravel())[0])
            bits = struct.unpack("<I", struct.pack("<f", float(fb.ravel()[flat])))[0]
            return BandResult(0, 0, 0, flat + self.y0 * self.width, bits, empty)
        if self.height == 0:
            return BandResult(0, 0, 0, NO_BAD, 0, empty)
        b = oracle.generate(self.st, fb, t_prev, t_now, log_eps=self.config.log_eps,
                            refractory_us=self.config.refractory_us, cap=self.cap if keep is None else keep)
        total = len(b) + b.dropped_count if keep is None else None
        b = oracle.canonical_sort(b)
        keys = pack_keys(torch.from_numpy(b.t.astype(np.int64)), torch.from_numpy(b.x.astype(np.int64)),
                         torch.from_numpy(b.y.astype(np.int64)) + self.y0, torch.from_numpy(b.polarity),
                         int(t_prev), KEY64_LAYOUT)
        return BandResult(total if total is not None else len(b), len(b), b.reservation_count, NO_BAD, 0, keys)


def host_merge(keys, counts):
    """Test stand-in for the evs_merge_runs kernel (CPU tensors over gloo): a
    stable sort of the bands' runs (key order is the canonical order)."""
    assert sum(counts) == keys.numel()
    return keys[np.argsort(keys.numpy(), kind="stable")]


def test_band_rows_partition_and_alignment():
    for H in (0, 1, 7, 30, 260, 720, 1080):
        for W in (1, 3, 37, 40, 346, 1280):
            for N in (1, 2, 3, 4, 8):
                rows = band_rows(H, W, N)
                assert len(rows) == N and rows[0][0] == 0 and rows[-1][1] == H
                for (a0, a1), (b0, b1) in zip(rows, rows[1:]):
                    assert a1 == b0
                for y0, y1 in rows:
                    assert 0 <= y0 <= y1 <= H and (y0 * W) % 32 == 0 or y0 == H


def test_plan_frame_capacity_and_bad():
    # totals 10, 5, 7 with cap 12: band0 keeps 10 (it held min(10, 12) = 10),
    # band1 may keep 2 (held 5: rerun), band2 none (held 7: rerun)
    p = plan_frame([[10, 10, 3, NO_BAD, 0], [5, 5, 2, NO_BAD, 0], [7, 7, 1, NO_BAD, 0]], 12)
    assert p.allowed == [10, 2, 0] and p.rerun == [1, 2]
    assert p.written == 12 and p.dropped == 10 and p.reservations == 6 and p.bad == NO_BAD
    p = plan_frame([[0, 0, 0, NO_BAD, 0], [0, 0, 0, 77, 5], [0, 0, 0, 40, 9]], 12)
    assert (p.bad, p.bad_bits) == (40, 9)
    p = plan_frame([[0, 0, 4, NO_BAD, 0]], 12)
    assert p.reservations == 0 and p.written == 0


def _sequence(W, H, n, seed):
    rng = np.random.default_rng(seed)
    return oracle.random_walk_sequence(rng, W, H, n)


def _worker(rank, world, port, q, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, H = 40, 30
        cap = {"normal": None, "capacity": 37, "bad": None}[case]
        cfg = EventCameraConfig(c_pos=0.12, c_neg=0.15, sigma_c=0.03, refractory_us=150,
                                max_events_per_frame=cap)
        frames = _sequence(W, H, 5, 3)
        full = oracle.init_state(frames[0], c_pos=0.12, c_neg=0.15, sigma_c=0.03, refractory_us=150, seed=4)
        ref_full = full.copy()
        rows = band_rows(H, W, world)
        band = OracleBand(full, rows[rank], cfg)
        cam = BandedCamera(band, TorchComm(), cfg, W, H, merge=host_merge)
        out = []
        for k in range(1, len(frames)):
            fr = frames[k].copy()
            if case == "bad" and k == 3:
                fr[20, 5] = np.nan   # row 20 lies in band 1
                fr[25, 1] = 2.0
                pre = (band.st.ref_log.copy(), band.st.last_event_t.copy())
                try:
                    cam.step(fr, (k - 1) * 1000, k * 1000)
                    out.append(("no-raise",))
                except ValueError as e:
                    out.append(("raised", str(e), np.array_equal(pre[0], band.st.ref_log),
                                np.array_equal(pre[1], band.st.last_event_t)))
                continue
            stats = AggregationStats()
            b = cam.step(fr, (k - 1) * 1000, k * 1000, stats=stats)
            exp = oracle.canonical_sort(oracle.generate(ref_full, frames[k], (k - 1) * 1000, k * 1000,
                                                        refractory_us=150, cap=cfg.capacity(W, H)))
            sl = slice(*rows[rank])
            state_ok = (np.array_equal(band.st.ref_log, ref_full.ref_log[sl])
                        and np.array_equal(band.st.last_event_t, ref_full.last_event_t[sl]))
            if rank == 0:
                ok = (b.same_events(exp) and b.dropped_count == exp.dropped_count
                      and stats.reservation_count == exp.reservation_count
                      and stats.events_emitted == len(exp))
                out.append(("frame", ok, state_ok, len(exp), exp.dropped_count))
            else:
                out.append(("frame", b is None, state_ok, len(exp), exp.dropped_count))
        q.put((rank, out))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, [("error", repr(e))]))
    finally:
        dist.destroy_process_group()


def _run(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = None
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, case)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("case", ["normal", "capacity"])
def test_banded_camera_two_ranks_matches_unsplit(case):
    res = _run(case)
    for rank in (0, 1):
        for item in res[rank]:
            assert item[0] == "frame", item
            assert item[1] and item[2], (rank, item)
    if case == "capacity":
        assert any(item[4] > 0 for item in res[0])  # the cut really happened
    assert sum(item[3] for item in res[0]) > 100


def test_banded_camera_bad_pixel_raises_everywhere_state_untouched():
    res = _run("bad")
    msgs = set()
    for rank in (0, 1):
        bad = [it for it in res[rank] if it[0] == "raised"]
        assert len(bad) == 1, res[rank]
        _, msg, ref_same, last_same = bad[0]
        assert ref_same and last_same
        msgs.add(msg)
        assert all(it[0] in ("frame", "raised") and (it[0] != "frame" or (it[1] and it[2])) for it in res[rank])
    assert msgs == {"invalid intensity np.float32(nan) at pixel (x=5, y=20)"}
