"""Multi-GPU plumbing: one process per GPU, independent camera streams per rank.

The event path has no data-path collective (pixels and streams are
independent), so scaling is by sharding streams across ranks.  NCCL is used
only when a consumer needs the events on one rank (BASELINE configs[4]):
``gather_keys`` is a gatherv built from an all_gather of the per-rank counts
(8 bytes per rank) plus grouped point-to-point sends into prefix offsets on
the destination (NCCL has no gatherv).  Events travel as packed keys written
on the device by the evs_pack_segments kernel: 4 bytes per event when the
sensor and the time span fit 31 bits (DAVIS: t_rel 12 + y 9 + x 9 + p 1),
else 8 (t_rel < 2^30 | y | x | p), instead of the 13-byte SoA.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_streams(num_streams: int, world_size: int, rank: int) -> list[int]:
    """Streams owned by `rank`: stream s -> rank floor(s * N / S) (contiguous blocks)."""
    return [s for s in range(num_streams) if (s * world_size) // num_streams == rank]


def key32_layout(width: int, height: int, span_us: int):
    """Bit widths (t_rel, y, x) of a 4-byte key t_rel << (yb + xb + 1) | y << (xb + 1)
    | x << 1 | p for a sensor and a time span (DAVIS events in
    4 bytes), or None when they need more than 31 bits (the key stays a
    non-negative int32, so its order is the canonical order)."""
    def bits(n):
        return max(1, int(n - 1).bit_length())
    tb, yb, xb = bits(span_us), bits(height), bits(width)
    return (tb, yb, xb) if tb + yb + xb + 1 <= 31 else None


KEY64_LAYOUT = (30, 16, 16)  # 8-byte keys: t_rel < 2^30 (the sign bit stays clear), 16-bit y and x


def pack_segments(counts, rows, t_base: int, layout, key_bytes: int, out=None, y_offset: int = 0):
    """Packed keys of an evs_step output (device [nseg][cap] SoA rows t, x, y, p
    and device per-segment counts) written back to back by the evs_pack_segments
    kernel.  Returns (keys, offsets[nseg + 1]) on the device, no host sync;
    ``out`` (a big enough 1-D int32 / int64 tensor) is reused when given;
    ``y_offset`` shifts a row band's rows to sensor rows."""
    from . import _lib

    t, x, y, p = rows
    nseg, cap = t.shape
    dt = torch.int32 if key_bytes == 4 else torch.int64
    if out is None or out.dtype != dt or out.numel() < nseg * cap:
        out = torch.empty(nseg * cap, dtype=dt, device=t.device)
    offs = torch.empty(nseg + 1, dtype=torch.int64, device=t.device)
    _, yb, xb = layout
    rc = _lib.load().evs_pack_segments(nseg, counts.data_ptr(), cap, t.data_ptr(), x.data_ptr(), y.data_ptr(),
                                       p.data_ptr(), int(t_base), int(y_offset), key_bytes, yb, xb, out.data_ptr(),
                                       offs.data_ptr(), out.numel(), _lib.stream_ptr())
    _lib.check(rc, "evs_pack_segments")
    return out, offs


def unpack_keys(k: torch.Tensor, t_base: int, layout):
    """Packed keys -> (t, x, y, p) tensors (consumer side; 4- or 8-byte keys)."""
    tb, yb, xb = layout
    k = k.to(torch.int64)
    t = (k >> (yb + xb + 1)) + t_base
    y = ((k >> (xb + 1)) & ((1 << yb) - 1)).to(torch.int32)
    x = ((k >> 1) & ((1 << xb) - 1)).to(torch.int32)
    p = torch.where((k & 1) == 1, 1, -1).to(torch.int8)
    return t, x, y, p


def pack_keys(t, x, y, p, t_base: int, layout):
    """SoA events -> packed keys with torch ops (tests and host-side callers; the
    step output is packed on the device by pack_segments).  Raises when a time
    does not fit the layout's t_rel bits."""
    tb, yb, xb = layout
    tr = (t.to(torch.int64) - t_base)
    if tr.numel() and (int(tr.min()) < 0 or int(tr.max()) >= (1 << tb)):
        raise ValueError(f"event times must lie in [t_base, t_base + 2**{tb})")
    k = (tr << (yb + xb + 1)) | ((y.to(torch.int64) & 0xFFFF) << (xb + 1)) | \
        ((x.to(torch.int64) & 0xFFFF) << 1) | (p > 0).to(torch.int64)
    return k.to(torch.int32) if tb + yb + xb + 1 <= 31 else k


def gather_events(t, x, y, p, t_base: int, width: int, height: int, span_us: int, dst: int = 0, group=None):
    """Gather every rank's events (SoA, times in [t_base, t_base + span_us)) to
    ``dst`` in rank order as packed keys: 4 bytes per event when the sensor and
    span fit in 31 bits (DAVIS: 12 + 9 + 9 + 1), else 8.  Returns (t, x, y, p)
    on dst, None elsewhere; the same layout decision on every rank."""
    lay = key32_layout(width, height, span_us) or KEY64_LAYOUT
    keys = pack_keys(t, x, y, p, t_base, lay)
    out, _ = gather_keys(keys, dst=dst, group=group)
    return None if out is None else unpack_keys(out, t_base, lay)


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
