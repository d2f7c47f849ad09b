"""Multi-GPU plumbing: one process per GPU, independent camera streams per rank.

The event path has no data-path collective (pixels and streams are
independent), so scaling is by sharding streams across ranks.  NCCL is used
only when a consumer needs the events on one rank (BASELINE configs[4]):
``gather_keys`` is a gatherv built from an all_gather of the per-rank counts
(8 bytes per rank) plus grouped point-to-point sends into prefix offsets on
the destination (NCCL has no gatherv).  Events travel as the packed 64-bit
keys the kernels already use (t_rel << 33 | y << 17 | x << 1 | p), 8 bytes
per event instead of the 13-byte SoA.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_streams(num_streams: int, world_size: int, rank: int) -> list[int]:
    """Streams owned by `rank`: stream s -> rank floor(s * N / S) (contiguous blocks)."""
    return [s for s in range(num_streams) if (s * world_size) // num_streams == rank]


def pack_keys(t: torch.Tensor, x: torch.Tensor, y: torch.Tensor, p: torch.Tensor, t_base: int) -> torch.Tensor:
    """SoA events -> packed int64 keys relative to t_base (t - t_base < 2**31)."""
    tr = (t - t_base).to(torch.int64)
    return (tr << 33) | ((y.to(torch.int64) & 0xFFFF) << 17) | ((x.to(torch.int64) & 0xFFFF) << 1) | \
        (p > 0).to(torch.int64)


def unpack_keys(k: torch.Tensor, t_base: int):
    t = (k >> 33) + t_base
    y = ((k >> 17) & 0xFFFF).to(torch.int32)
    x = ((k >> 1) & 0xFFFF).to(torch.int32)
    p = torch.where((k & 1) == 1, 1, -1).to(torch.int8)
    return t, x, y, p


def gather_keys(local: torch.Tensor, dst: int = 0, group=None):
    """Gatherv of 1-D int64 tensors to `dst`.  Returns (concatenated, counts) on
    dst and (None, counts) elsewhere.  Rank order is preserved."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = local.device
    n = torch.tensor([local.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    if rank == dst:
        out = torch.empty(sum(counts), dtype=local.dtype, device=dev)
        offs = [0]
        for c in counts:
            offs.append(offs[-1] + c)
        ops = []
        for r in range(world):
            if r == dst:
                out[offs[r]:offs[r + 1]].copy_(local)
            elif counts[r]:
                ops.append(dist.P2POp(dist.irecv, out[offs[r]:offs[r + 1]], r, group=group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return out, counts
    if counts[rank]:
        for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, local.contiguous(), dst, group=group)]):
            w.wait()
    return None, counts


def gather_fixed(local: torch.Tensor, dst: int = 0, group=None):
    """Gather equally-shaped tensors (e.g. per-stream histograms) to dst."""
    world = dist.get_world_size(group)
    if dist.get_rank(group) == dst:
        bufs = [torch.empty_like(local) for _ in range(world)]
        dist.gather(local, gather_list=bufs, dst=dst, group=group)
        return torch.stack(bufs)
    dist.gather(local, dst=dst, group=group)
    return None
