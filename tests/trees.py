"""Tiny trees with known analytic behaviour (ports of the reference's
tests/util.py:18-53, 86-96) built with this package."""
import math

import numpy as np

import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import hh

H000 = 1.0 / (math.sqrt(2.0) * math.pi)  # value of the constant HH basis


def const_payload(sigma, rgb, coeff_count, k):
    """Time-constant density and view/time-constant colour (util.py:18-24)."""
    row = np.zeros(2 * coeff_count + 3 * k, dtype=np.float32)
    row[0] = sigma  # bump bases column 0 is the constant column
    for ch in range(3):
        row[2 * coeff_count + ch] = math.log(rgb[ch] / (1.0 - rgb[ch])) / H000
    return row


def const_tree(voxels, depth, frames=4, coeff_count=3, n_max=1):
    """{(x, y, z): (sigma, (r, g, b))} (util.py:27-38)."""
    bases = vv.make_bump_bases(frames, coeff_count)
    k = hh.basis_count(n_max)
    coords = np.array(list(voxels.keys()), dtype=np.int64).reshape(-1, 3)
    data = np.stack([const_payload(s, c, coeff_count, k) for (s, c) in voxels.values()]) if voxels \
        else np.zeros((0, 2 * coeff_count + 3 * k), dtype=np.float32)
    return vv.VOctree.from_cells(coords, data, bases, n_max, depth=depth)


def random_payload_tree(rng, depth=2, fill=0.6, frames=4, coeff_count=3, n_max=2, sigma_scale=2.0):
    """Random occupied cells with smooth random payloads (util.py:41-53)."""
    res = 1 << depth
    coords = np.argwhere(rng.random((res, res, res)) < fill)
    k = hh.basis_count(n_max)
    data = rng.normal(scale=0.5, size=(len(coords), 2 * coeff_count + 3 * k))
    data[:, 0] = rng.uniform(0.2, sigma_scale, size=len(coords))
    return vv.VOctree.from_cells(coords, data.astype(np.float32), vv.make_bump_bases(frames, coeff_count), n_max,
                                 depth=depth)


def fine_march(sigma_fn, color_fn, t0, t1, steps=10_000):
    """Dense-step compositing oracle over [t0, t1] (util.py:86-96)."""
    ts = np.linspace(t0, t1, steps + 1)
    mid = 0.5 * (ts[:-1] + ts[1:])
    dt = np.diff(ts)
    sig = np.array([sigma_fn(t) for t in mid])
    col = np.array([color_fn(t) for t in mid])
    e = np.exp(-sig * dt)
    trans = np.concatenate([[1.0], np.cumprod(e)[:-1]])
    w = trans * (1.0 - e)
    return (w[:, None] * col).sum(axis=0), w.sum()
