"""Per-frame node masks (vv_launch_mask.cu): dark subtrees cut from image walks.

A leaf with sigma 0 contributes nothing to a render (kernels.py:556-559:
the reference `continue`s before touching T or the accumulators), so an
image render that skips dark leaves and all-dark subtrees must produce
bitwise the same pixels.  These tests force the masks on (VV_NODE_MASK=1)
and off (=0) and compare every image entry point bitwise, on trees where
many leaves are dark in some frames: sparse sigma weights of both signs,
the cfg3 motion generator, edited trees (masks disabled) and multi-frame
groups (one mask = union of the group's frames).  The stats / visit paths
must keep the reference's full walk whatever the setting.
"""

import numpy as np
import pytest

from oracle import oracle
import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import synthetic

pytestmark = pytest.mark.gpu


def _exact(a, b, what=""):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    b = b.cpu().numpy() if hasattr(b, "cpu") else np.asarray(b)
    assert a.shape == b.shape, what
    assert np.array_equal(a, b), f"{what}: {np.count_nonzero(a != b)} mismatches"


def _dark_tree(seed=3, depth=6, frames=8):
    """Random occupancy; sigma weights of both signs, so that whole regions
    go dark in some frames and light up in others."""
    rng = np.random.default_rng(seed)
    res = 1 << depth
    coords = np.argwhere(rng.random((res, res, res)) < 0.2)
    c, k = 6, 14
    data = rng.normal(scale=0.5, size=(len(coords), 2 * c + 3 * k)).astype(np.float32)
    x = coords[:, 0] / res
    data[:, 0] = 40.0 * np.sin(6.0 * x + 1.0)  # dark on alternate slabs
    data[:, 1:c] = rng.normal(scale=8.0, size=(len(coords), c - 1))
    return vv.VOctree.from_cells(coords, data, vv.make_bump_bases(frames, c), 2, depth=depth)


def _with(monkeypatch, flag, fn):
    monkeypatch.setenv("VV_NODE_MASK", flag)
    try:
        return fn()
    finally:
        monkeypatch.delenv("VV_NODE_MASK")


@pytest.mark.parametrize("mode", ["per_frame", "auto"])
def test_masked_render_bitwise(cuda, monkeypatch, mode):
    tree = _dark_tree()
    cam = vv.Camera.look_at([1.9, -0.6, 1.3], [0.5, 0.5, 0.5], width=96, height=80)
    opts = vv.RenderOptions(frame_slice=mode)
    for f in range(tree.frames):
        on = _with(monkeypatch, "1", lambda: vv.render(tree, cam, f, opts))
        off = _with(monkeypatch, "0", lambda: vv.render(tree, cam, f, opts))
        for a, b, n in zip((on.rgb, on.alpha, on.depth), (off.rgb, off.alpha, off.depth), "rad"):
            _exact(a, b, f"frame {f} {n}")
        cache_on = _with(monkeypatch, "1", lambda: vv.build_frame_cache(tree, f))
        img = vv.render(tree, cam, f, cache=cache_on)
        _exact(img.rgb, off.rgb, f"user cache frame {f}")


def test_masked_render_vs_oracle(cuda, monkeypatch):
    """Masked images against the oracle's full walk (counts from the same
    kernel's unmasked counting launch stay exact)."""
    tree = _dark_tree(seed=4)
    cam = vv.Camera.look_at([-0.8, 1.7, 1.6], [0.5, 0.5, 0.5], width=64, height=64)
    o, d = oracle.camera_rays(cam)
    for f in (0, 3, 6):
        img = _with(monkeypatch, "1", lambda: vv.render(tree, cam, f))
        ref = oracle.render_rays(tree, o, d, f)
        rgb, alpha, depth = oracle.finalize(ref["premult"], ref["alpha"], ref["tbar"])
        assert np.abs(img.rgb.reshape(-1, 3) - rgb).max() < 1e-4
        assert np.abs(img.alpha.reshape(-1) - alpha).max() < 1e-4
        assert ref["shaded"].sum() < ref["used"].sum()  # dark leaves were on the rays


def test_masked_playback_group_union(cuda, monkeypatch):
    """One mask per multi-frame group (union of the frames' lit subtrees):
    shared-walk playback bitwise equal to unmasked per-frame renders."""
    import torch

    tree = _dark_tree(seed=5)
    cam = vv.Camera.look_at([1.7, 1.5, -0.4], [0.5, 0.5, 0.5], width=80, height=64)
    h, w = cam.height, cam.width
    for frames in ([0, 1], [2, 5, 7], [1, 3, 4, 6]):
        outs = [(torch.empty((h, w, 3), device=cuda), torch.empty((h, w), device=cuda),
                 torch.empty((h, w), device=cuda)) for _ in frames]
        _with(monkeypatch, "1", lambda: vv.render_frames_into(tree, cam, frames, outs,
                                                               vv.RenderOptions(frame_slice="per_frame")))
        torch.cuda.synchronize()
        for f, o in zip(frames, outs):
            ref = _with(monkeypatch, "0", lambda: vv.render(tree, cam, f, vv.RenderOptions(frame_slice="per_frame")))
            _exact(o[0], ref.rgb, f"group {frames} frame {f} rgb")
            _exact(o[1], ref.alpha, f"group {frames} frame {f} alpha")
            _exact(o[2], ref.depth, f"group {frames} frame {f} depth")


def test_masked_render_rays_and_stats(cuda, monkeypatch):
    """render_rays without stats may walk the mask (same accumulators);
    with stats the counts stay the reference's full-walk counts."""
    tree = _dark_tree(seed=6, depth=5)
    rng = np.random.default_rng(2)
    o = rng.uniform(-1.0, 2.0, (3000, 3))
    d = rng.uniform(0.2, 0.8, (3000, 3)) - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    opts = vv.RenderOptions(frame_slice="per_frame")
    for f in (1, 4):
        on = _with(monkeypatch, "1", lambda: vv.render_rays(tree, o, d, f, opts))
        off = _with(monkeypatch, "0", lambda: vv.render_rays(tree, o, d, f, opts))
        for a, b in zip(on, off):
            _exact(a, b, f"rays frame {f}")
        st = _with(monkeypatch, "1", lambda: vv.render_rays(tree, o, d, f, opts, stats=True)[3])
        ref = oracle.render_rays(tree, o, d, f)
        _exact(st["sample_count"], ref["used"], "counts under masks")
        _exact(st["node_pops"], ref["pops"], "pops under masks")


def test_masked_scene_and_tiles(cuda, monkeypatch):
    """Scene instances with per-frame slices walk their masks; tile shards too."""
    import torch

    from paper_2202_06088_b200.distributed import TileRenderer

    tree = _dark_tree(seed=7)
    cam = vv.Camera.look_at([0.6, -2.5, 1.2], [0.6, 0.5, 0.5], width=96, height=64)
    scene = vv.Scene(instances=[
        vv.SceneInstance(name="a", tree=tree),
        vv.SceneInstance(name="b", tree=tree, affine=np.diag([0.8, 0.8, 0.8, 1.0]) @ np.eye(4),
                         timemap=vv.TimeMap.parse("shift(3)")),
    ])
    opts = vv.RenderOptions(frame_slice="per_frame")
    for g in (0, 2):
        on = _with(monkeypatch, "1", lambda: vv.render_scene(scene, cam, g, opts))
        off = _with(monkeypatch, "0", lambda: vv.render_scene(scene, cam, g, opts))
        _exact(on, off, f"scene g{g}")
    ref = _with(monkeypatch, "0", lambda: vv.render(tree, cam, 2, opts))
    slabs = []
    for s in range(3):
        tr = TileRenderer(96, 64, 32, rank=s, world=3, device=cuda)
        slabs.append(_with(monkeypatch, "1", lambda: tr.render_slab(tree, cam, 2, opts)).clone())
    tr.all.copy_(torch.stack(slabs))
    rgb = torch.empty((64, 96, 3), device=cuda)
    alpha = torch.empty((64, 96), device=cuda)
    depth = torch.empty((64, 96), device=cuda)
    tr.unpack(rgb, alpha, depth)
    torch.cuda.synchronize()
    _exact(rgb, ref.rgb, "tiles rgb")
    _exact(depth, ref.depth, "tiles depth")


def test_mask_disabled_for_edits_and_non_trees(cuda, monkeypatch):
    """Edits can light a dark leaf: edited trees never mask (bitwise equal to
    the unmasked render either way)."""
    tree = _dark_tree(seed=8, depth=4)
    tree.ensure_edit_arrays()
    tree.edit_rgb[::2, :3] = 0.3
    tree.edit_rgb[::2, 3] = 5.0  # density override on every other leaf
    tree.edit_t[::2] = (0, 7)
    cam = vv.Camera.look_at([1.8, 1.1, 1.4], [0.5, 0.5, 0.5], width=48, height=40)
    for f in (0, 5):
        on = _with(monkeypatch, "1", lambda: vv.render(tree, cam, f, vv.RenderOptions(frame_slice="per_frame")))
        ref = oracle.render_rays(tree, *oracle.camera_rays(cam), f)
        assert np.abs(on.alpha.reshape(-1) - ref["alpha"]).max() < 1e-4


def test_cfg3_masked_frames_bitwise(cuda):
    """cfg3 at 1080p: render() (auto: node masks on -- the motion tree is
    ~90% dark) bitwise equal to the unmasked counting launch."""
    import torch

    tree = synthetic.motion_tree()
    cam = synthetic.bench_camera()
    h, w = cam.height, cam.width
    for f in (3, 29, 58):
        img = vv.render(tree, cam, f)
        rgb = torch.empty((h, w, 3), device=cuda)
        alpha = torch.empty((h, w), device=cuda)
        depth = torch.empty((h, w), device=cuda)
        used = torch.empty((h, w), dtype=torch.int32, device=cuda)
        vv.render_into(tree, cam, f, rgb, alpha, depth, sample_count=used)
        torch.cuda.synchronize()
        _exact(img.rgb, rgb, f"cfg3 rgb {f}")
        _exact(img.alpha, alpha, f"cfg3 alpha {f}")
        _exact(img.depth, depth, f"cfg3 depth {f}")
