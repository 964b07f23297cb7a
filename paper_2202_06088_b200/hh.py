"""Hyperspherical-harmonic index bookkeeping needed by the render path.

Host-side restatement of the parts of the reference's ``voxvid.hh``
(pkg/src/voxvid/hh.py) that the renderer's API surface depends on: basis
counts, index orderings and the normalisation constants that feed
``kernels.basis_tables`` (kernels.py:56-76).  The evaluation itself runs
on the GPU (paper_2202_06088_b200/csrc/vv_device.cuh).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

__all__ = [
    "HHIndex",
    "BasisTruncation",
    "basis_count",
    "index_list",
    "sh_pair_list",
    "radial_pair_list",
    "double_factorial",
    "hh_norm",
    "sh_prefactor",
]


@dataclass(frozen=True)
class HHIndex:
    """Index triple of one HH basis element: 0 <= l <= n, -l <= m <= l (hh.py:53-65)."""

    n: int
    l: int
    m: int

    def __post_init__(self):
        if self.n < 0 or not (0 <= self.l <= self.n):
            raise ValueError(f"invalid HH index: need 0 <= l <= n, got n={self.n} l={self.l}")
        if abs(self.m) > self.l:
            raise ValueError(f"invalid HH index: need |m| <= l, got l={self.l} m={self.m}")


@dataclass(frozen=True)
class BasisTruncation:
    """Truncation at principal degree n_max (hh.py:88-104)."""

    n_max: int

    def __post_init__(self):
        if self.n_max < 0:
            raise ValueError(f"n_max must be non-negative, got {self.n_max}")

    @property
    def count(self) -> int:
        return basis_count(self.n_max)

    @property
    def sh_count(self) -> int:
        return (self.n_max + 1) ** 2


def basis_count(n_max: int) -> int:
    """K = sum_{n <= n_max} (n+1)^2 (hh.py:107-109)."""
    return sum((n + 1) ** 2 for n in range(n_max + 1))


@lru_cache(maxsize=None)
def index_list(n_max: int) -> tuple:
    """Kept indices, lexicographic by (n, l, m) (hh.py:112-120)."""
    return tuple(
        HHIndex(n, l, m) for n in range(n_max + 1) for l in range(n + 1) for m in range(-l, l + 1)
    )


@lru_cache(maxsize=None)
def sh_pair_list(l_max: int) -> tuple:
    return tuple((l, m) for l in range(l_max + 1) for m in range(-l, l + 1))


@lru_cache(maxsize=None)
def radial_pair_list(n_max: int) -> tuple:
    return tuple((n, l) for n in range(n_max + 1) for l in range(n + 1))


def double_factorial(k: int) -> float:
    out = 1.0
    while k > 1:
        out *= k
        k -= 2
    return out


@lru_cache(maxsize=None)
def hh_norm(n: int, l: int) -> float:
    """A_nl = (2l)!! sqrt(2(n+1)(n-l)! / (pi (n+l+1)!)) (hh.py:249-262)."""
    if not (0 <= l <= n):
        raise ValueError(f"need 0 <= l <= n, got n={n} l={l}")
    ratio = math.factorial(n - l) / math.factorial(n + l + 1)
    return double_factorial(2 * l) * math.sqrt(2.0 * (n + 1) * ratio / math.pi)


@lru_cache(maxsize=None)
def sh_prefactor(l: int, m: int) -> float:
    """Real-SH constant with the Condon-Shortley phase and sqrt(2) (hh.py:193-207)."""
    mu = abs(m)
    k = math.sqrt((2 * l + 1) / (4.0 * math.pi) * math.factorial(l - mu) / math.factorial(l + mu))
    pref = ((-1.0) ** mu) * k
    if mu > 0:
        pref *= math.sqrt(2.0)
    return pref
