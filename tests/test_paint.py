"""compose.paint (compose.py:482-532) on the GPU: termination voxels, edit
channels and skipped pixels against the reference (tests/golden/paint.npz),
plus the reference's behavioural paint tests (test_compose.py:328-386)."""
import math

import numpy as np
import pytest

from golden_util import camera_from, load, tree_from
from oracle import oracle
import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import hh
from paper_2202_06088_b200.compose import SceneInstance, duplicate, render_instance

H000 = 1.0 / (math.sqrt(2.0) * math.pi)  # constant HH basis value (reference tests/util.py:11)


def _const_tree(voxels, depth, frames=4, coeff_count=3, n_max=1):
    """Time-constant density/colour voxels (reference tests/util.py:18-38)."""
    bases = vv.make_bump_bases(frames, coeff_count)
    k = hh.basis_count(n_max)
    rows = []
    for sigma, rgb in voxels.values():
        row = np.zeros(2 * coeff_count + 3 * k, dtype=np.float32)
        row[0] = sigma
        for ch in range(3):
            row[2 * coeff_count + ch] = math.log(rgb[ch] / (1.0 - rgb[ch])) / H000
        rows.append(row)
    coords = np.array(list(voxels.keys()), dtype=np.int64).reshape(-1, 3)
    return vv.VOctree.from_cells(coords, np.stack(rows), bases, n_max, depth=depth)


def _wall():
    return _const_tree({(0, y, z): (800.0, (0.4, 0.4, 0.4)) for y in range(2) for z in range(2)}, depth=1)


def test_paint_bad_time_range():
    tree = _wall()
    cam = vv.Camera.look_at([-2.0, 0.5, 0.5], [0.25, 0.5, 0.5], width=4, height=4)
    with pytest.raises(ValueError, match="time range"):
        vv.paint(tree, cam, np.array([[0, 0]]), (1, 0, 0), (0, 99))


@pytest.mark.gpu
def test_termination_leaves_bit_exact(cuda):
    g = load("paint")
    tree = tree_from(g)
    got = vv.termination_leaves(tree, g["origins"], g["dirs"], 1, 0.9)
    assert np.array_equal(got, g["term_leaf"])
    assert np.array_equal(got, oracle.termination_leaves(tree, g["origins"], g["dirs"], 1, 0.9))


@pytest.mark.gpu
def test_paint_matches_reference(cuda):
    g = load("paint")
    tree = tree_from(g)
    cam = camera_from(g)
    before = vv.render(tree, cam, 2)  # a cached replica exists: edits must reach it in place
    res = vv.paint(tree, cam, g["p1_mask"], (0.9, 0.2, 0.1), (1, 4), alpha_threshold=0.9)
    assert res["edited_voxels"] == int(g["p1_edited"])
    assert np.array_equal(np.array(res["skipped_pixels"], np.int64).reshape(-1, 2), g["p1_skipped"])
    assert np.array_equal(tree.edit_rgb, g["p1_edit_rgb"]) and np.array_equal(tree.edit_t, g["p1_edit_t"])
    res = vv.paint(tree, cam, g["p2_pixels"], (0.1, 0.8, 0.3), (2, 5), alpha_threshold=0.5, target_density=7.5,
                   frame=3)
    assert res["edited_voxels"] == int(g["p2_edited"])
    assert np.array_equal(np.array(res["skipped_pixels"], np.int64).reshape(-1, 2), g["p2_skipped"])
    assert np.array_equal(tree.edit_rgb, g["p2_edit_rgb"]) and np.array_equal(tree.edit_t, g["p2_edit_t"])
    # the in-place edit push renders exactly like a fresh upload of the edited tree
    after = vv.render(tree, cam, 2)
    fresh = tree_from(g)
    fresh.edit_rgb, fresh.edit_t = tree.edit_rgb.copy(), tree.edit_t.copy()
    ref = vv.render(fresh, cam, 2)
    assert np.array_equal(after.rgb, ref.rgb) and np.array_equal(after.alpha, ref.alpha)
    assert not np.array_equal(after.rgb, before.rgb)


@pytest.mark.gpu
def test_paint_empty_space_skips(cuda):
    tree = _const_tree({(0, 0, 0): (5.0, (0.5, 0.5, 0.5))}, depth=1)
    cam = vv.Camera.look_at([-2.0, 0.8, 0.8], [0.9, 0.8, 0.8], width=8, height=8)
    res = vv.paint(tree, cam, np.array([[0, 0], [1, 0]]), (1.0, 0.0, 0.0), (0, 3))
    assert res["edited_voxels"] == 0
    assert len(res["skipped_pixels"]) == 2
    assert not tree.has_edits


@pytest.mark.gpu
def test_paint_opaque_wall_view_consistent(cuda):
    tree = _wall()
    cam_a = vv.Camera.look_at([-2.0, 0.5, 0.5], [0.25, 0.5, 0.5], width=16, height=16)
    cam_b = vv.Camera.look_at([-1.5, 1.5, 0.6], [0.25, 0.5, 0.5], width=16, height=16)
    before_b0 = vv.render(tree, cam_b, 0)
    before_b3 = vv.render(tree, cam_b, 3)
    mask = np.zeros((16, 16), dtype=bool)
    mask[6:10, 6:10] = True
    res = vv.paint(tree, cam_a, mask, (1.0, 0.05, 0.05), (0, 2))
    assert res["edited_voxels"] >= 1
    assert res["skipped_pixels"] == []
    after_b0 = vv.render(tree, cam_b, 0)
    assert (after_b0.rgb[..., 0] - before_b0.rgb[..., 0]).max() > 0.3
    after_b3 = vv.render(tree, cam_b, 3)  # outside the painted range: untouched
    np.testing.assert_array_equal(after_b3.rgb, before_b3.rgb)


@pytest.mark.gpu
def test_paint_shared_across_duplicates(cuda):
    tree = _wall()
    a = SceneInstance(name="a", tree=tree)
    b = duplicate(a, "b")
    cam = vv.Camera.look_at([-2.0, 0.5, 0.5], [0.25, 0.5, 0.5], width=8, height=8)
    img_before = render_instance(b, cam, 0)
    vv.paint(a.tree, cam, np.ones((8, 8), dtype=bool), (0.0, 1.0, 0.0), (0, 3))
    img_after = render_instance(b, cam, 0)
    assert (np.asarray(img_after.rgb)[..., 1] - np.asarray(img_before.rgb)[..., 1]).max() > 0.3
