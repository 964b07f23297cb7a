"""Deterministic synthetic VOctrees and cameras for the BASELINE.json configs.

The reference ships no VOctree synthesiser; SURVEY.md section 8(d) defines
the generator every benchmark and parity case uses:

* occupancy: cell (x, y, z) in [0, 2^d)^3 with centre c = (i + 0.5)/2^d - 0.5
  is occupied iff | |c| - 0.30 | <= (12/512)/2 (a spherical performer shell,
  12 voxels thick at depth 9); rows in lexicographic (x, y, z) order;
* payload: rng = default_rng(seed); data = normal(0, 0.3, (n, 2C+3K)) as
  float32; data[:, 0] = uniform(200 s, 800 s) with s = 2^(d-9);
  data[:, 1:C] *= 0.01; bases = make_bump_bases(T, C), C = 31;
* camera: look_at((1.6, 1.3, 0.9), (0.5, 0.5, 0.5), up z, focal 1.08 max(W, H)).

Config 3 (motion-heavy), 4 (four placed performers) and 5 (stereo) follow
the same table.  Everything here is host-side input generation.
"""

from __future__ import annotations

import math

import numpy as np

from . import hh
from .octree import VOctree
from .render import Camera
from .temporal import TemporalBases, make_bump_bases

__all__ = ["shell_coords", "shell_tree", "motion_tree", "bench_camera", "scene_config4", "stereo_cameras", "CONFIGS"]

C_DEFAULT = 31


def shell_coords(depth: int, radius: float = 0.30, thickness: float = 12.0 / 512.0) -> np.ndarray:
    """Occupied cells of the spherical shell, lexicographic (np.argwhere order)."""
    res = 1 << depth
    c = (np.arange(res, dtype=np.float64) + 0.5) / res - 0.5
    out = []
    cy, cz = np.meshgrid(c, c, indexing="ij")
    ryz = cy * cy + cz * cz
    for i in range(res):
        r = np.sqrt(c[i] * c[i] + ryz)
        yz = np.argwhere(np.abs(r - radius) <= thickness / 2.0)
        if len(yz):
            out.append(np.concatenate([np.full((len(yz), 1), i, dtype=np.int64), yz], axis=1))
    return np.concatenate(out, axis=0) if out else np.zeros((0, 3), dtype=np.int64)


def shell_tree(depth: int = 9, n_max: int = 2, frames: int = 30, seed: int = 0, coeff_count: int = C_DEFAULT):
    """Config 1/2 generator."""
    coords = shell_coords(depth)
    n = len(coords)
    k = hh.basis_count(n_max)
    rng = np.random.default_rng(seed)
    data = rng.normal(0.0, 0.3, (n, 2 * coeff_count + 3 * k)).astype(np.float32)
    s = 2.0 ** (depth - 9)
    data[:, 0] = rng.uniform(200.0 * s, 800.0 * s, n)
    data[:, 1:coeff_count] *= 0.01
    bases = make_bump_bases(frames, coeff_count)
    return VOctree.from_cells(coords, data, bases, n_max, depth=depth)


def motion_tree(depth: int = 9, n_max: int = 2, frames: int = 60, seed: int = 0, coeff_count: int = C_DEFAULT):
    """Config 3: per-voxel density bump selected by azimuth, learned-looking B."""
    coords = shell_coords(depth)
    n = len(coords)
    k = hh.basis_count(n_max)
    rng = np.random.default_rng(seed)
    data = rng.normal(0.0, 0.3, (n, 2 * coeff_count + 3 * k)).astype(np.float32)
    data[:, :coeff_count] = 0.0
    res = 1 << depth
    cx = (coords[:, 0] + 0.5) / res - 0.5
    cy = (coords[:, 1] + 0.5) / res - 0.5
    phi = np.arctan2(cy, cx)
    j = 1 + (np.floor((phi + math.pi) / (2 * math.pi) * 30).astype(np.int64) % 30)
    data[np.arange(n), j] = rng.uniform(200.0, 800.0, n)
    a = make_bump_bases(frames, coeff_count).a.astype(np.float64)
    b = a + rng.normal(0.0, 0.1, (frames, coeff_count))
    return VOctree.from_cells(coords, data, TemporalBases(a, b), n_max, depth=depth)


def bench_camera(width: int = 1920, height: int = 1080) -> Camera:
    return Camera.look_at(eye=(1.6, 1.3, 0.9), target=(0.5, 0.5, 0.5), up=(0.0, 0.0, 1.0), width=width,
                          height=height, focal=1.08 * max(width, height))


def _rz(a):
    m = np.eye(4)
    m[0, 0] = math.cos(a)
    m[0, 1] = -math.sin(a)
    m[1, 0] = math.sin(a)
    m[1, 1] = math.cos(a)
    return m


def _tr(x, y, z):
    m = np.eye(4)
    m[:3, 3] = [x, y, z]
    return m


def scene_config4(trees, width: int = 1920, height: int = 1080):
    """Config 4: 4 placed performers with time offsets."""
    from .compose import Scene, SceneInstance, TimeMap

    c = np.array([0.5, 0.5, 0.5])
    inst = []
    for i, tree in enumerate(trees):
        s = np.eye(4)
        if i == 3:
            s[:3, :3] *= 0.8
        aff = _tr(1.1 * (i - 1.5), 0.0, 0.0) @ _tr(*c) @ _rz(0.5 * i) @ s @ _tr(*(-c))
        inst.append(SceneInstance(name=f"performer{i}", tree=tree, affine=aff,
                                  timemap=TimeMap.parse(f"shift({3 * i})|loop(30)")))
    cam = Camera.look_at(eye=(0.5, -3.0, 1.4), target=(0.5, 0.5, 0.5), up=(0.0, 0.0, 1.0), width=width,
                         height=height, focal=0.75 * width)
    return Scene(instances=inst), cam


def stereo_cameras(size: int = 2160, baseline: float = 0.032):
    """Config 5: two eyes at eye +- baseline*right, both looking at the target."""
    eye = np.array([1.6, 1.3, 0.9])
    target = np.array([0.5, 0.5, 0.5])
    mono = Camera.look_at(eye, target, width=size, height=size, focal=1.08 * size)
    right = mono.c2w[:3, 0]
    return [Camera.look_at(eye + sgn * baseline * right, target, width=size, height=size, focal=1.08 * size)
            for sgn in (-1.0, 1.0)]


CONFIGS = {
    1: dict(depth=7, n_max=1, frames=16, width=64, height=64, frame=5),
    2: dict(depth=9, n_max=2, frames=30, width=1920, height=1080),
    3: dict(depth=9, n_max=2, frames=60, width=1920, height=1080),
}
