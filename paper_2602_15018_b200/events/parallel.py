"""Chunk-parallel aggregation API: drop-in mirror of ``evsim.events.parallel``.

Reference: /root/reference/pkg/src/evsim/events/parallel.py.

On the B200 the reference's "32-lane chunk claims one block via a locked
cursor" becomes: each warp covers 32-pixel chunks (a ``__ballot_sync`` mask
per chunk, parallel.py:79-99), a block-wide scan places every lane's
variable-length output, and a decoupled-lookback prefix across tiles gives
each tile its global base -- no per-chunk atomics and a deterministic,
pixel-major placement (identical to the serial definition, so capacity
drops are exactly the serial ones).  ``generate_events_parallel`` then
returns the batch already in canonical (t, y, x, p) order (a fused stable
radix pass on t), which the reference only guarantees after
``canonical_sort``.

``ReservationCursor`` / ``reserve_block`` / ``compute_chunk_mask`` are the
reference's host-side instrumentation objects, kept for API parity.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from .. import _lib
from .model import run_generate
from .types import DeviceEventBatch, EventBatch, EventCameraConfig, IntensityFrame, PixelStateGrid

CHUNK_WIDTH = 32  # parallel.py:32


class ReservationCursor:
    """parallel.py:47-71: bump allocator over a bounded buffer."""

    def __init__(self, capacity: int):
        self.capacity = capacity
        self.next_free = 0
        self.reservation_count = 0
        self._lock = threading.Lock()

    def reserve(self, count: int) -> tuple[int, int]:
        if count < 0:
            raise ValueError("reservation count must be >= 0")
        if count == 0:
            return self.next_free, 0
        with self._lock:
            base = self.next_free
            self.next_free = base + count
            self.reservation_count += 1
        granted = min(base + count, self.capacity) - base
        return base, max(granted, 0)


def reserve_block(cursor: ReservationCursor, count: int) -> tuple[int, int]:
    """parallel.py:74-76."""
    return cursor.reserve(count)


@dataclass
class ChunkMask:
    """parallel.py:79-88: ballot mask of event-producing lanes plus counts."""

    bits: int
    counts: np.ndarray

    @property
    def popcount(self) -> int:
        return bin(self.bits).count("1")


def compute_chunk_mask(counts: np.ndarray) -> ChunkMask:
    """parallel.py:91-99 (the host analogue of __ballot_sync(count > 0))."""
    if len(counts) > CHUNK_WIDTH:
        raise ValueError(f"a chunk has at most {CHUNK_WIDTH} lanes")
    c = np.asarray(counts)
    bits = int(np.sum((c > 0).astype(np.uint64) << np.arange(len(c), dtype=np.uint64))) if len(c) else 0
    return ChunkMask(bits=bits, counts=c)


@dataclass
class AggregationStats:
    """parallel.py:102-109: per-frame instrumentation."""

    reservation_count: int = 0
    events_emitted: int = 0
    collect_spans: bool = False
    write_spans: list[tuple[int, int]] = field(default_factory=list)


def canonical_sort(batch):
    """parallel.py:112-123: order by (t, y, x, polarity) ascending, stable; drops kept.

    Runs as LSD onesweep radix passes on the GPU (evs_canonical_sort).  Host
    batches come back as host batches, device batches stay on the device.
    """
    from ..represent import canonical_sort as _cs

    return _cs(batch)


def generate_events_parallel(
    state: PixelStateGrid,
    frame: IntensityFrame,
    t_prev: int,
    t_now: int,
    config: EventCameraConfig,
    workers: int = 1,
    stats: AggregationStats | None = None,
    device_output: bool = False,
):
    """parallel.py:126-273 on the GPU; output already in canonical order.

    ``workers`` is accepted for API parity (validated like the reference,
    parallel.py:142-143) but the GPU ignores it.  ``device_output=True``
    returns a DeviceEventBatch that stays in HBM.
    """
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return run_generate(state, frame, t_prev, t_now, config, _lib.EVS_ORDER_CANONICAL, stats,
                        device_output=device_output)
