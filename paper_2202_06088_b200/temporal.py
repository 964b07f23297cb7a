"""Temporal bases and payload-layout helpers (host side).

Restates the parts of the reference's ``voxvid.temporal``
(pkg/src/voxvid/temporal.py) that define the VOctree payload the renderer
consumes: the shared (T, C) basis matrices A/B (temporal.py:53-79), the
payload length 2C+3K (temporal.py:128-129), the bump-basis initialiser
(temporal.py:207-226) and the edit channels (temporal.py:82-102).  The
per-sample decodes (density relu(A w), hyper angle pi*sigmoid(B w), HH
colour) run on the GPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

__all__ = [
    "TemporalBases",
    "EditChannels",
    "CoefficientVector",
    "payload_length",
    "n_max_for_count",
    "make_bump_bases",
]


@dataclass
class TemporalBases:
    """Shared basis matrices A (density) and B (hyper angle), both (T, C) float32."""

    a: np.ndarray
    b: np.ndarray

    def __post_init__(self):
        self.a = np.ascontiguousarray(self.a, dtype=np.float32)
        self.b = np.ascontiguousarray(self.b, dtype=np.float32)
        if self.a.ndim != 2 or self.a.shape != self.b.shape:
            raise ValueError(f"A and B must share a (T, C) shape, got {self.a.shape} vs {self.b.shape}")

    @property
    def frames(self) -> int:
        return self.a.shape[0]

    @property
    def count(self) -> int:
        return self.a.shape[1]

    def copy(self) -> "TemporalBases":
        return TemporalBases(self.a.copy(), self.b.copy())


@dataclass
class EditChannels:
    """Appearance-edit payload of a painted voxel (temporal.py:82-102)."""

    target_rgb: tuple
    time_range: tuple
    target_density: float | None = None

    def __post_init__(self):
        if any(not (0.0 <= c <= 1.0) for c in self.target_rgb):
            raise ValueError(f"edit rgb out of [0,1]: {self.target_rgb}")
        if self.target_density is not None and self.target_density < 0:
            raise ValueError(f"edit density must be non-negative: {self.target_density}")

    @property
    def active(self) -> bool:
        return self.time_range[0] <= self.time_range[1]


@dataclass
class CoefficientVector:
    """One voxel's payload (temporal.py:105-125)."""

    w_sigma: np.ndarray
    w_gamma: np.ndarray
    w_hh: np.ndarray
    edit: EditChannels | None = None

    def __post_init__(self):
        self.w_sigma = np.asarray(self.w_sigma, dtype=np.float64)
        self.w_gamma = np.asarray(self.w_gamma, dtype=np.float64)
        self.w_hh = np.asarray(self.w_hh, dtype=np.float64)
        if self.w_sigma.shape != self.w_gamma.shape or self.w_sigma.ndim != 1:
            raise ValueError("w_sigma and w_gamma must be equal-length vectors")
        if self.w_hh.ndim != 2 or self.w_hh.shape[1] != 3:
            raise ValueError(f"w_hh must be (K, 3), got {self.w_hh.shape}")


def payload_length(c: int, k: int, with_edit: bool = False) -> int:
    return 2 * c + 3 * k + (5 if with_edit else 0)


@lru_cache(maxsize=None)
def n_max_for_count(k: int) -> int:
    """Invert K = sum (n+1)^2 (temporal.py:132-141)."""
    n, total = 0, 1
    while total < k:
        n += 1
        total += (n + 1) ** 2
    if total != k:
        raise ValueError(f"{k} is not a valid truncated basis count")
    return n


def make_bump_bases(frames: int, count: int) -> TemporalBases:
    """Constant column plus shifted raised cosines (temporal.py:207-226)."""
    if frames < 1 or count < 1:
        raise ValueError("need frames >= 1 and count >= 1")
    a = np.zeros((frames, count), dtype=np.float64)
    a[:, 0] = 1.0
    t = np.arange(frames, dtype=np.float64)
    n_bumps = count - 1
    if n_bumps > 0:
        centers = np.linspace(0.0, frames - 1.0, n_bumps) if n_bumps > 1 else [0.5 * (frames - 1)]
        width = max(1.0, 1.4 * (frames - 1) / max(1, n_bumps - 1))
        for j, c in enumerate(centers):
            d = np.abs(t - c)
            a[:, j + 1] = np.where(d < width, 0.5 * (1.0 + np.cos(math.pi * d / width)), 0.0)
    return TemporalBases(a, a.copy())
