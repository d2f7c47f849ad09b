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


def key32_layout(width: int, height: int, span_us: int):
    """Bit widths (t_rel, y, x) of a 4-byte key t_rel << (yb + xb + 1) | y << (xb + 1)
    | x << 1 | p for a sensor and a time span (DAVIS events in
    4 bytes), or None when they need more than 31 bits (the key stays a
    non-negative int32, so its order is the canonical order)."""
    def bits(n):
        return max(1, int(n - 1).bit_length())
    tb, yb, xb = bits(span_us), bits(height), bits(width)
    return (tb, yb, xb) if tb + yb + xb + 1 <= 31 else None


def pack_keys32(t: torch.Tensor, x: torch.Tensor, y: torch.Tensor, p: torch.Tensor, t_base: int,
                layout) -> torch.Tensor:
    """SoA events -> int32 keys (layout from key32_layout; 0 <= t - t_base < 2**tb)."""
    tb, yb, xb = layout
    tr = (t - t_base).to(torch.int64)
    k = (tr << (yb + xb + 1)) | ((y.to(torch.int64) & 0xFFFF) << (xb + 1)) | \
        ((x.to(torch.int64) & 0xFFFF) << 1) | (p > 0).to(torch.int64)
    return k.to(torch.int32)


def unpack_keys32(k: torch.Tensor, t_base: int, layout):
    tb, yb, xb = layout
    k = k.to(torch.int64)
    t = (k >> (yb + xb + 1)) + t_base
    y = ((k >> (xb + 1)) & ((1 << yb) - 1)).to(torch.int32)
    x = ((k >> 1) & ((1 << xb) - 1)).to(torch.int32)
    p = torch.where((k & 1) == 1, 1, -1).to(torch.int8)
    return t, x, y, p


def gather_events(t, x, y, p, t_base: int, width: int, height: int, span_us: int, dst: int = 0, group=None):
    """Gather every rank's events (SoA, times in [t_base, t_base + span_us)) to
    ``dst`` in rank order as packed keys: 4 bytes per event when the sensor and
    span fit in 31 bits (DAVIS: 12 + 9 + 9 + 1), else 8.  Returns (t, x, y, p)
    on dst, None elsewhere; the same layout decision on every rank."""
    lay = key32_layout(width, height, span_us)
    if lay is None:
        keys = pack_keys(t, x, y, p, t_base)
        out, _ = gather_keys(keys, dst=dst, group=group)
        return None if out is None else unpack_keys(out, t_base)
    keys = pack_keys32(t, x, y, p, t_base, lay)
    out, _ = gather_keys(keys, dst=dst, group=group)
    return None if out is None else unpack_keys32(out, t_base, lay)


def gather_keys(local: torch.Tensor, dst: int = 0, group=None):
    """Gatherv of 1-D int64 / int32 tensors to `dst`.  Returns (concatenated, counts) on
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
