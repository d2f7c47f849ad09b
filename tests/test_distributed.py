"""Multi-process (gloo, world_size 2, CPU) tests of the stream sharding and the
gatherv used to collect packed events on one rank."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_15018_b200.distributed import (KEY64_LAYOUT, gather_events, gather_fixed, gather_keys, key32_layout,
                                               pack_keys, shard_streams, unpack_keys)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r owns streams shard_streams(8, 2, r) and produces r*3+1 events per stream
        mine = shard_streams(8, world, rank)
        t = torch.arange(len(mine) * (rank * 3 + 1), dtype=torch.int64) + 1000
        x = torch.full_like(t, rank + 1).to(torch.int16)
        y = torch.full_like(t, 7).to(torch.int16)
        p = torch.where(t % 2 == 0, 1, -1).to(torch.int8)
        keys = pack_keys(t, x, y, p, 1000, KEY64_LAYOUT)
        out, counts = gather_keys(keys, dst=0)
        hist = torch.full((3, 4), rank, dtype=torch.int64)
        stacked = gather_fixed(hist, dst=0)
        # DAVIS-sized events travel as 4-byte keys, HD ones with a long span as 8-byte keys
        ev = []
        for W, H, span in ((346, 260, 4000), (1280, 720, 1 << 20)):
            n = 50 + 30 * rank
            g = torch.Generator().manual_seed(rank)
            tt = torch.randint(0, span, (n,), generator=g) + 7000
            xx = torch.randint(0, W, (n,), generator=g).to(torch.int16)
            yy = torch.randint(0, H, (n,), generator=g).to(torch.int16)
            pp = (torch.randint(0, 2, (n,), generator=g) * 2 - 1).to(torch.int8)
            got = gather_events(tt, xx, yy, pp, 7000, W, H, span, dst=0)
            ev.append((tt.tolist(), xx.tolist(), yy.tolist(), pp.tolist(),
                       None if got is None else [v.tolist() for v in got]))
        if rank == 0:
            q.put(("ok", counts, out.tolist(), stacked.tolist(), ev))
        else:
            q.put(("r1", ev))
    finally:
        dist.destroy_process_group()


def test_shard_streams_partition():
    for S in (1, 7, 64, 256):
        for N in (1, 2, 4, 8):
            owned = [shard_streams(S, N, r) for r in range(N)]
            flat = sorted(s for o in owned for s in o)
            assert flat == list(range(S))
            sizes = [len(o) for o in owned]
            assert max(sizes) - min(sizes) <= 1


def test_pack_unpack_roundtrip():
    t = torch.tensor([5, 6, 1999], dtype=torch.int64) + 10**9
    x = torch.tensor([0, 345, 1279], dtype=torch.int16)
    y = torch.tensor([0, 259, 719], dtype=torch.int16)
    p = torch.tensor([1, -1, 1], dtype=torch.int8)
    t2, x2, y2, p2 = unpack_keys(pack_keys(t, x, y, p, 10**9, KEY64_LAYOUT), 10**9, KEY64_LAYOUT)
    assert torch.equal(t2, t) and torch.equal(x2, x.to(torch.int32)) and torch.equal(y2, y.to(torch.int32))
    assert torch.equal(p2, p)
    # 8-byte keys stay non-negative: t - t_base must be < 2^30 (ADVICE: no sign-bit overflow)
    with pytest.raises(ValueError):
        pack_keys(t + (1 << 30), x, y, p, 10**9, KEY64_LAYOUT)
    with pytest.raises(ValueError):
        pack_keys(t - 10, x, y, p, 10**9, KEY64_LAYOUT)


@pytest.mark.timeout(120)
def test_gatherv_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict((r[0], r) for r in (q.get(timeout=100), q.get(timeout=100)))
    for pr in procs:
        pr.join(timeout=60)
    res, r1 = got["ok"], got["r1"]
    counts, out, stacked = res[1], res[2], res[3]
    for (t0, x0, y0, p0, merged), (t1, x1, y1, p1, _none) in zip(res[4], r1[1]):
        t, x, y, p = merged
        assert t == t0 + t1 and p == p0 + p1
        assert x == [v & 0xFFFF for v in x0 + x1] and y == [v & 0xFFFF for v in y0 + y1]
    assert counts == [4 * 1, 4 * 4]
    keys = torch.tensor(out)
    t, x, y, p = unpack_keys(keys, 1000, KEY64_LAYOUT)
    # rank order preserved: rank 0's events first
    assert x[:4].tolist() == [1] * 4 and x[4:].tolist() == [2] * 16
    assert t[:4].tolist() == [1000, 1001, 1002, 1003]
    assert stacked[0][0][0] == 0 and stacked[1][2][3] == 1


def test_key32_layout_roundtrip_and_order():
    assert key32_layout(346, 260, 4000) == (12, 9, 9)
    assert key32_layout(1280, 720, 50_000) is None
    lay = key32_layout(640, 480, 2000)
    g = torch.Generator().manual_seed(3)
    n = 5000
    t = torch.randint(0, 2000, (n,), generator=g) + 10**9
    x = torch.randint(0, 640, (n,), generator=g).to(torch.int16)
    y = torch.randint(0, 480, (n,), generator=g).to(torch.int16)
    p = (torch.randint(0, 2, (n,), generator=g) * 2 - 1).to(torch.int8)
    k = pack_keys(t, x, y, p, 10**9, lay)
    assert k.dtype == torch.int32 and int(k.min()) >= 0
    t2, x2, y2, p2 = unpack_keys(k, 10**9, lay)
    assert torch.equal(t2, t) and torch.equal(x2, x.to(torch.int32)) and torch.equal(y2, y.to(torch.int32))
    assert torch.equal(p2, p)
    # int32 key order == the 8-byte key order == canonical (t, y, x, p)
    assert torch.equal(torch.argsort(k, stable=True),
                       torch.argsort(pack_keys(t, x, y, p, 10**9, KEY64_LAYOUT), stable=True))
