"""The NCCL gather of packed event keys (BASELINE config 5) between 2 GPUs:
collected whenever the box has >= 2 GPUs (tests/conftest.py deselects it on
one-GPU boxes, which every GPU call of this build had; the same logic runs
over gloo in tests/test_distributed.py)."""

import os
import socket

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2602_15018_b200 import events as ev
    from paper_2602_15018_b200.distributed import gather_keys, key32_layout, pack_segments, shard_streams, unpack_keys
    from paper_2602_15018_b200.simulator import EventSimulator
    from paper_2602_15018_b200.synth import texture_frame

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        W, H, S, T = 346, 260, 6, 4
        mine = shard_streams(S, world, rank)
        sim = EventSimulator(W, H, streams=len(mine), frames_per_step=T, config=ev.EventCameraConfig(), device=dev)
        sim.reset([texture_frame(W, H, 0.137 * s) for s in mine], seeds=mine)
        frames = np.stack([[texture_frame(W, H, 0.137 * s + 0.02 * (f + 1)) for f in range(T)] for s in mine])
        sim.step(torch.from_numpy(frames).to(dev))
        r = sim.result()
        e = sim.engine
        lay = key32_layout(W, H, T * 1000)
        keys, offs = pack_segments(e.info[0], (e.ev_t, e.ev_x, e.ev_y, e.ev_p), 0, lay, 4)
        n = int(offs[-1].item())
        out, counts = gather_keys(keys[:n], dst=0)
        if rank == 0:
            t, x, y, p = unpack_keys(out, 0, lay)
            q.put(("ok", counts, t.cpu().numpy(), x.cpu().numpy(), y.cpu().numpy(), p.cpu().numpy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_nccl_gather_of_packed_keys_two_gpus():
    import torch
    import torch.multiprocessing as mp

    import oracle
    from paper_2602_15018_b200.synth import texture_frame

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
    _, counts, t, x, y, p = res
    # rank order = stream order; every stream's T canonical segments back to back
    W, H, S, T = 346, 260, 6, 4
    exp = []
    for s in range(S):
        st = oracle.init_state(texture_frame(W, H, 0.137 * s), seed=s)
        for f in range(T):
            exp.append(oracle.canonical_sort(oracle.generate(st, texture_frame(W, H, 0.137 * s + 0.02 * (f + 1)),
                                                             f * 1000, (f + 1) * 1000)))
    et = np.concatenate([b.t.astype(np.int64) for b in exp])
    assert sum(counts) == len(et) == len(t)
    assert np.array_equal(t, et)
    assert np.array_equal(x, np.concatenate([b.x for b in exp]).astype(np.int32))
    assert np.array_equal(y, np.concatenate([b.y for b in exp]).astype(np.int32))
    assert np.array_equal(p, np.concatenate([b.polarity for b in exp]))
