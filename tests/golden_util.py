"""Helpers to rebuild golden-case trees (tests/golden/*.npz) as package VOctrees."""

from pathlib import Path

import numpy as np

from paper_2202_06088_b200.octree import VOctree
from paper_2202_06088_b200.render import Camera
from paper_2202_06088_b200.temporal import TemporalBases

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def tree_from(g, prefix="tree_"):
    er = g.get(prefix + "edit_rgb")
    et = g.get(prefix + "edit_t")
    return VOctree(
        int(g[prefix + "depth"]), g[prefix + "node_child"], g[prefix + "leaf_coords"], g[prefix + "leaf_data"],
        TemporalBases(g[prefix + "a"], g[prefix + "b"]), int(g[prefix + "n_max"]), g[prefix + "bbox_lo"],
        float(g[prefix + "side"]),
        edit_rgb=None if er is None else er.copy(), edit_t=None if et is None else et.copy(),
    )


def camera_from(g, prefix="cam_"):
    w, h = (int(v) for v in g[prefix + "wh"])
    fx, fy, cx, cy = (float(v) for v in g[prefix + "f"])
    return Camera(w, h, fx, fy, cx, cy, g[prefix + "c2w"])
