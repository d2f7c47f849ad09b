"""Synthetic moving-texture input (the reference's own benchmark workload).

``texture_frame`` restates ``_texture_frame`` (events_bench.py:19-26): a
drifting diagonal sinusoid computed in f64 and stored as f32, so every pixel
changes every frame.  With the reference drift of 0.02 per frame the texture
is periodic over 50 frames, which lets benchmarks cycle a pre-uploaded ring
of frames without a discontinuity.
"""

from __future__ import annotations

import numpy as np

PERIOD_FRAMES = 50  # phase drift 0.02/frame -> period 1.0


def texture_frame(width: int, height: int, phase: float) -> np.ndarray:
    x = np.arange(width) / width
    y = np.arange(height) / height
    grid = np.add.outer(y * 2.0, x * 3.0)
    return (0.5 + 0.45 * np.sin(2.0 * np.pi * (grid + phase))).astype(np.float32)


def texture_ring(width: int, height: int, frames: int, drift: float = 0.02, phase0: float = 0.0,
                 device=None):
    """[frames, H, W] f32 ring, frame k at phase phase0 + k*drift, on `device` (torch)."""
    import torch

    out = torch.empty((frames, height, width), dtype=torch.float32, device=device)
    for k in range(frames):
        out[k].copy_(torch.from_numpy(texture_frame(width, height, phase0 + k * drift)))
    return out


def stream_phase(s: int) -> float:
    """Per-stream phase offset for multi-camera workloads."""
    return 0.137 * s
