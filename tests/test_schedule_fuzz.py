"""Randomised cross-check of every round-2 scheduling and skipping path:
camera plans (persistent warps, cost order, cached coverage), occupied-box
rectangles, node masks, region culling, playback plans, banded host copies.
None of them may change a pixel: each render is compared bitwise with the
plain static per-sample render of the same tree, camera and frame, over
random trees (depth 3-7, n_max 0-3, sparse and dense, with and without
edits) and random cameras (outside, grazing, inside the cube)."""

import numpy as np
import pytest

import paper_2202_06088_b200 as vv
from paper_2202_06088_b200.distributed import band_plan, pixel_costs, render_region

pytestmark = pytest.mark.gpu


def _eq(a, b, what):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    b = b.cpu().numpy() if hasattr(b, "cpu") else np.asarray(b)
    assert np.array_equal(a, b), f"{what}: {np.count_nonzero(a != b)} mismatches"


def _tree(rng, depth, n_max, edits):
    res = 1 << depth
    fill = rng.uniform(0.03, 0.6)
    coords = np.argwhere(rng.random((res, res, res)) < fill)
    c = int(rng.integers(3, 9))
    k = (n_max + 1) * (n_max + 2) * (2 * n_max + 3) // 6
    data = rng.normal(scale=0.5, size=(len(coords), 2 * c + 3 * k)).astype(np.float32)
    data[:, 0] = rng.uniform(-20.0, 60.0, len(coords))  # some leaves dark in some frames
    data[:, 1:c] = rng.normal(scale=10.0, size=(len(coords), c - 1))
    lo = tuple(rng.uniform(-0.5, 0.5, 3))
    side = float(rng.choice([1.0, 0.5, 2.0, 1.3]))
    tree = vv.VOctree.from_cells(coords, data, vv.make_bump_bases(6, c), n_max, bbox_lo=lo, side=side, depth=depth)
    if edits:
        tree.ensure_edit_arrays()
        sel = rng.choice(tree.n_leaves, size=max(1, tree.n_leaves // 5), replace=False)
        tree.edit_rgb[sel, :3] = rng.uniform(0, 1, (len(sel), 3))
        tree.edit_rgb[sel, 3] = np.where(rng.random(len(sel)) < 0.5, -1.0, rng.uniform(0, 8, len(sel)))
        tree.edit_t[sel] = (1, 4)
    return tree


def _camera(rng, tree, w, h):
    c = np.asarray(tree.bbox_lo) + 0.5 * tree.side
    kind = rng.integers(3)
    if kind == 0:  # outside
        eye = c + tree.side * rng.uniform(1.2, 2.5) * rng.normal(size=3) / 1.0
    elif kind == 1:  # grazing: far, narrow
        eye = c + tree.side * 4.0 * rng.normal(size=3)
    else:  # inside the cube
        eye = c + tree.side * rng.uniform(-0.3, 0.3, 3)
    tgt = c + tree.side * rng.uniform(-0.3, 0.3, 3)
    if np.linalg.norm(tgt - eye) < 1e-3:
        tgt = eye + np.array([0.3, 0.2, 0.1])
    focal = float(rng.uniform(0.5, 3.0)) * max(w, h)
    return vv.Camera.look_at(eye, tgt, width=w, height=h, focal=focal)


@pytest.mark.parametrize("seed", range(12))
def test_schedules_bitwise(cuda, seed, monkeypatch):
    import torch

    rng = np.random.default_rng(1000 + seed)
    depth = int(rng.integers(3, 8))
    n_max = int(rng.integers(0, 4))
    tree = _tree(rng, depth, n_max, edits=bool(seed % 4 == 3))
    w, h = int(rng.choice([64, 80, 97])), int(rng.choice([48, 56, 71]))
    plan = vv.CameraPlan(cuda)
    mplan_frames = [0, 2, 5]
    for _ in range(3):
        cam = _camera(rng, tree, w, h)
        for f in (0, 2, 5):
            ref = vv.render(tree, cam, f, vv.RenderOptions(frame_slice="per_sample"), out="torch")
            for mask, vis in (("0", "0"), ("1", "0"), ("0", "1"), ("1", "1")):
                monkeypatch.setenv("VV_NODE_MASK", mask)
                monkeypatch.setenv("VV_VISIBLE", vis)
                for mode in ("per_frame", "auto"):
                    opts = vv.RenderOptions(frame_slice=mode)
                    out = [torch.empty((h, w, 3), device=cuda), torch.empty((h, w), device=cuda),
                           torch.empty((h, w), device=cuda)]
                    vv.render_into(tree, cam, f, *out, opts, plan=plan)
                    torch.cuda.synchronize()
                    _eq(out[0], ref.rgb, f"plan rgb mask{mask} {mode} f{f}")
                    _eq(out[1], ref.alpha, f"plan alpha mask{mask} {mode} f{f}")
                    _eq(out[2], ref.depth, f"plan depth mask{mask} {mode} f{f}")
                host = vv.render(tree, cam, f)  # banded host copies, stream plan
                _eq(host.rgb, ref.rgb, f"host rgb mask{mask} f{f}")
                _eq(host.depth, ref.depth, f"host depth mask{mask} f{f}")
            monkeypatch.delenv("VV_NODE_MASK")
            monkeypatch.delenv("VV_VISIBLE")
        # regions (culled slices) and playback
        costs = pixel_costs(tree, cam, 0)
        edges = band_plan(costs.sum(dim=1).cpu().numpy(), int(rng.integers(2, 5)))
        rgb = torch.full((h, w, 3), float("nan"), device=cuda)
        alpha = torch.full((h, w), float("nan"), device=cuda)
        depth = torch.full((h, w), float("nan"), device=cuda)
        for k in range(len(edges) - 1):
            render_region(tree, cam, 2, (0, edges[k], w, edges[k + 1]), rgb, alpha, depth,
                          vv.RenderOptions(frame_slice="per_frame"), plan=vv.CameraPlan(cuda))
        ref = vv.render(tree, cam, 2, vv.RenderOptions(frame_slice="per_sample"), out="torch")
        torch.cuda.synchronize()
        _eq(rgb, ref.rgb, "regions rgb")
        _eq(depth, ref.depth, "regions depth")
        outs = [(torch.empty((h, w, 3), device=cuda), torch.empty((h, w), device=cuda),
                 torch.empty((h, w), device=cuda)) for _ in mplan_frames]
        vv.render_frames_into(tree, cam, mplan_frames, outs, vv.RenderOptions(frame_slice="per_frame"))
        torch.cuda.synchronize()
        for f, o in zip(mplan_frames, outs):
            ref = vv.render(tree, cam, f, vv.RenderOptions(frame_slice="per_sample"), out="torch")
            _eq(o[0], ref.rgb, f"playback rgb f{f}")
            _eq(o[2], ref.depth, f"playback depth f{f}")
