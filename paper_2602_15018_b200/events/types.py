"""Event-camera data types: drop-in mirror of ``evsim.events.types``.

Reference: /root/reference/pkg/src/evsim/events/types.py.  Names, fields,
defaults and validation messages are the reference's.  Differences are in
residency only:

* ``PixelStateGrid`` keeps its arrays resident on the GPU (torch tensors in
  HBM); the reference attribute names still return host numpy arrays
  (copies) so reference-style code and tests keep working.
* ``EventBatch`` is the reference's host SoA batch (numpy, same dtypes).
  ``DeviceEventBatch`` is the same SoA kept in HBM for the batched path.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterator, NamedTuple

import numpy as np

# types.py:17 -- effective thresholds are clamped to this floor
MIN_THRESHOLD = 0.01
# types.py:22 -- crossing tolerance absorbing float32 state rounding
CROSSING_TOL = 1e-4


class Event(NamedTuple):
    """types.py:25-31."""

    t: int
    x: int
    y: int
    polarity: int


@dataclass
class EventBatch:
    """types.py:34-79: host SoA batch plus the count dropped by capacity limits."""

    t: np.ndarray  # uint64, microseconds
    x: np.ndarray  # uint16
    y: np.ndarray  # uint16
    polarity: np.ndarray  # int8, +1 or -1
    dropped_count: int = 0
    # True when the batch is known to be in canonical (t, y, x, p) order
    canonical: bool = field(default=False, repr=False, compare=False)
    # the inputs of concat_batches (lets canonical_sort merge instead of sort)
    parts: list | None = field(default=None, repr=False, compare=False)

    @staticmethod
    def empty(dropped_count: int = 0) -> "EventBatch":
        return EventBatch(
            t=np.empty(0, np.uint64), x=np.empty(0, np.uint16), y=np.empty(0, np.uint16),
            polarity=np.empty(0, np.int8), dropped_count=dropped_count, canonical=True,
        )

    @staticmethod
    def from_events(events: list[Event], dropped_count: int = 0) -> "EventBatch":
        return EventBatch(
            t=np.array([e.t for e in events], np.uint64),
            x=np.array([e.x for e in events], np.uint16),
            y=np.array([e.y for e in events], np.uint16),
            polarity=np.array([e.polarity for e in events], np.int8),
            dropped_count=dropped_count,
        )

    def __len__(self) -> int:
        return len(self.t)

    def __iter__(self) -> Iterator[Event]:
        for i in range(len(self.t)):
            yield Event(int(self.t[i]), int(self.x[i]), int(self.y[i]), int(self.polarity[i]))

    def same_events(self, other: "EventBatch") -> bool:
        """types.py:71-79: exact, order-sensitive equality."""
        return (
            len(self) == len(other)
            and bool(np.array_equal(self.t, other.t))
            and bool(np.array_equal(self.x, other.x))
            and bool(np.array_equal(self.y, other.y))
            and bool(np.array_equal(self.polarity, other.polarity))
        )

    def to_device(self, device=None) -> "DeviceEventBatch":
        import torch

        dev = device or torch.device("cuda", torch.cuda.current_device())
        return DeviceEventBatch(
            t=torch.from_numpy(np.ascontiguousarray(self.t).view(np.int64)).to(dev),
            x=torch.from_numpy(np.ascontiguousarray(self.x).view(np.int16)).to(dev),
            y=torch.from_numpy(np.ascontiguousarray(self.y).view(np.int16)).to(dev),
            polarity=torch.from_numpy(np.ascontiguousarray(self.polarity)).to(dev),
            dropped_count=self.dropped_count, canonical=self.canonical,
        )


@dataclass
class DeviceEventBatch:
    """EventBatch resident in HBM.

    ``t`` is int64 holding the reference's uint64 microseconds; ``x``/``y``
    are int16 tensors holding uint16 bits; ``polarity`` is int8.
    """

    t: "object"
    x: "object"
    y: "object"
    polarity: "object"
    dropped_count: int = 0
    canonical: bool = False
    parts: list | None = None

    def __len__(self) -> int:
        return int(self.t.shape[0])

    def to_host(self) -> EventBatch:
        return EventBatch(
            t=self.t.cpu().numpy().view(np.uint64),
            x=self.x.cpu().numpy().view(np.uint16),
            y=self.y.cpu().numpy().view(np.uint16),
            polarity=self.polarity.cpu().numpy(),
            dropped_count=int(self.dropped_count), canonical=self.canonical,
        )

    def same_events(self, other) -> bool:
        return self.to_host().same_events(other.to_host() if isinstance(other, DeviceEventBatch) else other)


def concat_batches(batches: list) -> EventBatch:
    """types.py:82-92: concatenate in order; dropped counts add."""
    if not batches:
        return EventBatch.empty()
    if all(isinstance(b, DeviceEventBatch) for b in batches):
        import torch

        return DeviceEventBatch(
            t=torch.cat([b.t for b in batches]), x=torch.cat([b.x for b in batches]),
            y=torch.cat([b.y for b in batches]), polarity=torch.cat([b.polarity for b in batches]),
            dropped_count=sum(int(b.dropped_count) for b in batches), parts=list(batches),
        )
    hs = [b.to_host() if isinstance(b, DeviceEventBatch) else b for b in batches]
    return EventBatch(
        t=np.concatenate([b.t for b in hs]), x=np.concatenate([b.x for b in hs]),
        y=np.concatenate([b.y for b in hs]), polarity=np.concatenate([b.polarity for b in hs]),
        dropped_count=sum(b.dropped_count for b in hs), parts=list(hs),
    )


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


@dataclass
class IntensityFrame:
    """types.py:95-109.  ``values`` may also be a float32 CUDA tensor (H, W)."""

    width: int
    height: int
    t: int
    values: "np.ndarray"

    def __post_init__(self) -> None:
        if _is_torch(self.values):
            import torch

            if self.values.dtype != torch.float32:
                self.values = self.values.to(torch.float32)
            shape = tuple(self.values.shape)
        else:
            self.values = np.asarray(self.values, np.float32)
            shape = self.values.shape
        if shape != (self.height, self.width):
            raise ValueError(
                f"frame values shape {shape} != (height={self.height}, width={self.width})"
            )


@dataclass
class DepthFrame:
    """types.py:112-126."""

    width: int
    height: int
    t: int
    values: np.ndarray

    def __post_init__(self) -> None:
        self.values = np.asarray(self.values, np.float32)
        if self.values.shape != (self.height, self.width):
            raise ValueError(
                f"depth values shape {self.values.shape} != (height={self.height}, width={self.width})"
            )


@dataclass
class EventCameraConfig:
    """types.py:129-156: contrast-threshold sensor parameters."""

    c_pos: float = 0.2
    c_neg: float = 0.2
    sigma_c: float = 0.0
    refractory_us: int = 0
    log_eps: float = 0.01
    noise_rate_hz: float = 0.0
    max_events_per_frame: int | None = None  # None -> 8 * width * height

    def __post_init__(self) -> None:
        if self.c_pos <= 0 or self.c_neg <= 0:
            raise ValueError("contrast thresholds must be positive")
        if self.log_eps <= 0:
            raise ValueError("log_eps must be positive")
        if self.refractory_us < 0:
            raise ValueError("refractory_us must be >= 0")
        if self.noise_rate_hz < 0:
            raise ValueError("noise_rate_hz must be >= 0")
        if self.sigma_c < 0:
            raise ValueError("sigma_c must be >= 0")

    def capacity(self, width: int, height: int) -> int:
        if self.max_events_per_frame is not None:
            return self.max_events_per_frame
        return 8 * width * height


class PixelStateGrid:
    """types.py:159-178, resident in HBM.

    Device tensors: ``d_ref_log`` (f32), ``d_last_event_t`` (i64),
    ``d_thresholds_pos`` / ``d_thresholds_neg`` (f32), all (H, W).  When
    both threshold grids are constant (sigma_c == 0) the kernels read the
    scalar instead of the grids (``uniform_thresholds``).
    """

    def __init__(self, width: int, height: int, ref_log, last_event_t, thresholds_pos,
                 thresholds_neg, device=None):
        import torch

        self.width = int(width)
        self.height = int(height)
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.device = dev

        def up(a, dt_np, dt_t):
            if _is_torch(a):
                return a.to(device=dev, dtype=dt_t).reshape(self.height, self.width).contiguous()
            arr = np.ascontiguousarray(np.asarray(a, dt_np).reshape(self.height, self.width))
            return torch.from_numpy(arr).to(dev)

        self.d_ref_log = up(ref_log, np.float32, torch.float32)
        self.d_last_event_t = up(last_event_t, np.int64, torch.int64)
        self.d_thresholds_pos = up(thresholds_pos, np.float32, torch.float32)
        self.d_thresholds_neg = up(thresholds_neg, np.float32, torch.float32)
        self.uniform_thresholds = None
        hp = thresholds_pos if not _is_torch(thresholds_pos) else None
        hn = thresholds_neg if not _is_torch(thresholds_neg) else None
        if hp is not None and hn is not None:
            hp = np.asarray(hp, np.float32).ravel()
            hn = np.asarray(hn, np.float32).ravel()
            if hp.size and np.all(hp == hp[0]) and np.all(hn == hn[0]):
                self.uniform_thresholds = (float(hp[0]), float(hn[0]))
        self._ctx = {}

    # Reference attribute names -> READ-ONLY host snapshots of the HBM state (an
    # in-place edit such as ``state.ref_log[mask] = v`` raises instead of being
    # silently lost); assign the whole attribute to write: ``state.ref_log = a``.
    @staticmethod
    def _snapshot(t) -> np.ndarray:
        a = t.cpu().numpy()
        a.flags.writeable = False
        return a

    @property
    def ref_log(self) -> np.ndarray:
        return self._snapshot(self.d_ref_log)

    @ref_log.setter
    def ref_log(self, v) -> None:
        self.d_ref_log.copy_(_as_tensor(v, self.d_ref_log))

    @property
    def last_event_t(self) -> np.ndarray:
        return self._snapshot(self.d_last_event_t)

    @last_event_t.setter
    def last_event_t(self, v) -> None:
        self.d_last_event_t.copy_(_as_tensor(v, self.d_last_event_t))

    @property
    def thresholds_pos(self) -> np.ndarray:
        return self._snapshot(self.d_thresholds_pos)

    @thresholds_pos.setter
    def thresholds_pos(self, v) -> None:
        self.d_thresholds_pos.copy_(_as_tensor(v, self.d_thresholds_pos))
        self._refresh_uniform()

    @property
    def thresholds_neg(self) -> np.ndarray:
        return self._snapshot(self.d_thresholds_neg)

    @thresholds_neg.setter
    def thresholds_neg(self, v) -> None:
        self.d_thresholds_neg.copy_(_as_tensor(v, self.d_thresholds_neg))
        self._refresh_uniform()

    def _refresh_uniform(self) -> None:
        """Thresholds changed: constant grids let the kernels read one scalar."""
        hp = self.d_thresholds_pos.reshape(-1)
        hn = self.d_thresholds_neg.reshape(-1)
        if hp.numel() and bool((hp == hp[0]).all()) and bool((hn == hn[0]).all()):
            self.uniform_thresholds = (float(hp[0].item()), float(hn[0].item()))
        else:
            self.uniform_thresholds = None

    def copy(self) -> "PixelStateGrid":
        c = PixelStateGrid.__new__(PixelStateGrid)
        c.width, c.height, c.device = self.width, self.height, self.device
        c.d_ref_log = self.d_ref_log.clone()
        c.d_last_event_t = self.d_last_event_t.clone()
        c.d_thresholds_pos = self.d_thresholds_pos.clone()
        c.d_thresholds_neg = self.d_thresholds_neg.clone()
        c.uniform_thresholds = self.uniform_thresholds
        c._ctx = {}
        return c

    def __repr__(self) -> str:
        return f"PixelStateGrid(width={self.width}, height={self.height}, device={self.device})"


def _as_tensor(v, like):
    import torch

    if _is_torch(v):
        return v.to(device=like.device, dtype=like.dtype).reshape(like.shape)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(v).astype(
        np.float32 if like.dtype == torch.float32 else np.int64)).reshape(tuple(like.shape))).to(like.device)
