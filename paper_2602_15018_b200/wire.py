"""Events wire encoding straight from the event buffers.

The step after the hot path in ``SimNode._publish_bundle``
(/root/reference/pkg/src/evsim/sim/orchestrator.py:191-200) serializes the
canonical batch with the ``Events`` schema (sim/schemas.py:13-15,42-46) and
wraps it in a Cortex wire frame (messaging/frame.py:1-46).  This module writes
the same bytes directly: header fields on the host, and for a device batch the
event arrays are DMA'd from HBM straight to their offsets in one pinned frame
buffer (no intermediate host copies).

Layout (little-endian), byte-identical to ``frame_encode(topic, hash, ns,
serialize(events_values(step_id, t_us, batch), EVENTS_SCHEMA))``:
  u8 topic length | topic | "CTX1" u8 version=1 u8 flags u16 0 | u64 schema hash |
  u64 publish ns | u64 payload length | payload
  payload: u64 step_id | u64 t_us | u64 dropped | for t(u64), x(u16), y(u16),
  polarity(i8): u8 dtype code, u8 rank=1, u32 length, raw array bytes
  (schema.py:194-225; dtype codes = 1-based index in SCALAR_KINDS, schema.py:27-30).
"""

from __future__ import annotations

import struct

import numpy as np

EVENTS_DECLARATION = "Events{step_id:u64;t_us:u64;dropped:u64;t:u64[*];x:u16[*];y:u16[*];polarity:i8[*]}"
_SCALAR_KINDS = ("u8", "u16", "u32", "u64", "i8", "i16", "i32", "i64", "f32", "f64", "bool")  # schema.py:27
_CODE = {k: i + 1 for i, k in enumerate(_SCALAR_KINDS)}
_FIELDS = (("t", "u64", np.dtype("<u8")), ("x", "u16", np.dtype("<u2")), ("y", "u16", np.dtype("<u2")),
           ("polarity", "i8", np.dtype("<i1")))
_HEADER = struct.Struct("<4sBBHQQQ")  # frame.py:25
MAGIC = b"CTX1"
VERSION = 1


def fnv1a64(data: bytes) -> int:
    """schema.py:157-163."""
    h = 0xCBF29CE484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


EVENTS_SCHEMA_HASH = fnv1a64(EVENTS_DECLARATION.encode("utf-8"))  # schema.py:166-168 (0xf0300ed12c62f35d)


def events_payload_size(counts) -> int:
    """Exact payload bytes for arrays of lengths (n_t, n_x, n_y, n_p) (schema.py:277-295)."""
    return 24 + sum(6 + n * dt.itemsize for n, (_nm, _k, dt) in zip(counts, _FIELDS))


def _layout(topic: str, counts):
    traw = topic.encode("utf-8")
    if len(traw) > 255:
        raise ValueError(f"topic exceeds 255 UTF-8 bytes: {topic!r}")  # frame.py:40-41
    head = 1 + len(traw) + _HEADER.size
    offs = []
    o = head + 24
    for n, (_nm, _k, dt) in zip(counts, _FIELDS):
        offs.append(o + 6)
        o += 6 + n * dt.itemsize
    return traw, head, offs, o


def _write_headers(buf: np.ndarray, traw: bytes, head: int, offs, counts, step_id, t_us, dropped,
                   publish_time_ns, flags) -> None:
    payload_len = offs[-1] + counts[-1] * _FIELDS[-1][2].itemsize - head
    mv = memoryview(buf)
    mv[0] = len(traw)
    mv[1:1 + len(traw)] = traw
    _HEADER.pack_into(mv, 1 + len(traw), MAGIC, VERSION, flags, 0, EVENTS_SCHEMA_HASH, int(publish_time_ns),
                      payload_len)
    struct.pack_into("<QQQ", mv, head, int(step_id) & 0xFFFFFFFFFFFFFFFF, int(t_us) & 0xFFFFFFFFFFFFFFFF,
                     int(dropped) & 0xFFFFFFFFFFFFFFFF)
    for (_nm, kind, _dt), off, n in zip(_FIELDS, offs, counts):
        struct.pack_into("<BBI", mv, off - 6, _CODE[kind], 1, n)


def encode_events_frame(topic: str, publish_time_ns: int, step_id: int, t_us: int, batch, flags: int = 0,
                        pool=None) -> np.ndarray:
    """Wire frame (uint8 array) of one Events message for a host EventBatch, a
    DeviceEventBatch, or a mapping with keys t, x, y, polarity, dropped.

    Device batches are copied from HBM directly into the frame (a pinned block
    from ``pool``, a runtime.PinnedPool); the result is then a view into it."""
    if isinstance(batch, dict):
        arrays = [batch[nm] for nm, _k, _dt in _FIELDS]
        dropped = batch["dropped"]
    else:
        arrays = [batch.t, batch.x, batch.y, batch.polarity]
        dropped = batch.dropped_count
    device = type(arrays[0]).__module__.startswith("torch") and arrays[0].is_cuda
    counts = [int(a.numel() if device else np.asarray(a).size) for a in arrays]
    traw, head, offs, total = _layout(topic, counts)
    if device:
        import torch

        from .runtime import PinnedPool

        pool = pool if pool is not None else _default_pool()
        t, root = pool.take(total)
        buf = root[:total]
        for a, off, n, (_nm, _k, dt) in zip(arrays, offs, counts, _FIELDS):
            if n:
                # raw bytes (the frame offsets are not element-aligned)
                t[off:off + n * dt.itemsize].copy_(a.contiguous().view(torch.uint8), non_blocking=True)
        _write_headers(buf, traw, head, offs, counts, step_id, t_us, dropped, publish_time_ns, flags)
        torch.cuda.current_stream().synchronize()
        return buf
    buf = np.empty(total, np.uint8)
    _write_headers(buf, traw, head, offs, counts, step_id, t_us, dropped, publish_time_ns, flags)
    for a, off, n, (_nm, _k, dt) in zip(arrays, offs, counts, _FIELDS):
        if n:
            # np.ascontiguousarray(value, dtype) as in schema._as_array (wrapping casts)
            buf[off:off + n * dt.itemsize] = np.ascontiguousarray(np.asarray(a).astype(dt, copy=False)).view(
                np.uint8)
    return buf


_POOL = None


def _default_pool():
    global _POOL
    if _POOL is None:
        from .runtime import PinnedPool

        _POOL = PinnedPool()
    return _POOL

