"""Multi-process (gloo, world_size 2, CPU) tests of the stream sharding and the
gatherv used to collect packed events on one rank."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_15018_b200.distributed import gather_fixed, gather_keys, pack_keys, shard_streams, unpack_keys


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
        keys = pack_keys(t, x, y, p, 1000)
        out, counts = gather_keys(keys, dst=0)
        hist = torch.full((3, 4), rank, dtype=torch.int64)
        stacked = gather_fixed(hist, dst=0)
        if rank == 0:
            q.put(("ok", counts, out.tolist(), stacked.tolist()))
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
    t2, x2, y2, p2 = unpack_keys(pack_keys(t, x, y, p, 10**9), 10**9)
    assert torch.equal(t2, t) and torch.equal(x2, x.to(torch.int32)) and torch.equal(y2, y.to(torch.int32))
    assert torch.equal(p2, p)


@pytest.mark.timeout(120)
def test_gatherv_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=100)
    for pr in procs:
        pr.join(timeout=60)
    assert res[0] == "ok"
    counts, out, stacked = res[1], res[2], res[3]
    assert counts == [4 * 1, 4 * 4]
    keys = torch.tensor(out)
    t, x, y, p = unpack_keys(keys, 1000)
    # rank order preserved: rank 0's events first
    assert x[:4].tolist() == [1] * 4 and x[4:].tolist() == [2] * 16
    assert t[:4].tolist() == [1000, 1001, 1002, 1003]
    assert stacked[0][0][0] == 0 and stacked[1][2][3] == 1
