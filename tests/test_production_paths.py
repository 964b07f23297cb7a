"""Parity of the kernel instantiations the BASELINE configs actually run.

Every production kernel choice is compared against the oracle (or the
reference's own golden vectors) at the size the bench runs it:

* cfg2 (depth-9 shell, 1080p): the sliced camera kernel with the regular
  segment queue -- per-pixel sample counts from the production
  instantiation bit-exact, images within 1e-4, on the FULL frame;
* cfg3 (motion tree, ~90% of leaves dark, 1080p): the same with the
  threshold-8 long-queue instantiations the tree's dark fraction selects
  (vv_launch_camera.cu, vv_launch_multi.cu), for render(), the shared-walk
  playback (render_frames_into / render_sequence) and the per-sample path;
* cfg4 (4 performers, one non-rigid): the reference's compose.render_scene
  golden through the lean per-sample scene kernel (k_render_scene_lean) and
  the sliced one (k_render_scene);
* cfg5 (2160^2 stereo): one eye full frame vs the oracle, and the 8-shard
  direct tile render bitwise equal to render().

Camera rays: the kernels generate rays in a fixed fp64 order; the oracle's
``camera_rays`` restates that order, so visits and counts compare
bit-exactly.  ``test_camera_ray_agreement`` measures how often those rays
visit exactly the same leaves as the reference's own BLAS-built
``Camera.rays``.

Contract (BASELINE.json north_star): visited leaves and per-ray sample
counts bit-exact; RGB/alpha/depth within 1e-4 absolute.
"""

import numpy as np
import pytest

from golden_util import camera_from, load
from oracle import oracle
import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import synthetic

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _exact(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    bad = np.count_nonzero(a != b)
    assert bad == 0, f"{what}: {bad} mismatches of {a.size}"


def _camera_render(tree, cam, frame, opts=vv.RenderOptions()):
    """render_into with per-pixel sample counts from the same kernel launch."""
    import torch

    h, w = cam.height, cam.width
    rgb = torch.empty((h, w, 3), dtype=torch.float32, device="cuda")
    alpha = torch.empty((h, w), dtype=torch.float32, device="cuda")
    depth = torch.empty((h, w), dtype=torch.float32, device="cuda")
    used = torch.full((h, w), -1, dtype=torch.int32, device="cuda")
    vv.render_into(tree, cam, frame, rgb, alpha, depth, opts, sample_count=used)
    torch.cuda.synchronize()
    return rgb.cpu().numpy(), alpha.cpu().numpy(), depth.cpu().numpy(), used.cpu().numpy()


def _check_images(rgb, alpha, depth, ref, idx=None, what=""):
    """Images vs the oracle's finalize_layer of its raw accumulators."""
    r_rgb, r_alpha, r_depth = oracle.finalize(ref["premult"], ref["alpha"], ref["tbar"])
    rgb = rgb.reshape(-1, 3)
    alpha = alpha.reshape(-1)
    depth = depth.reshape(-1)
    if idx is not None:
        rgb, alpha, depth = rgb[idx], alpha[idx], depth[idx]
    assert np.abs(rgb - r_rgb).max() < TOL, what
    assert np.abs(alpha - r_alpha).max() < TOL, what
    hit = r_alpha >= 1e-3
    assert np.abs(depth[hit] - r_depth[hit]).max() < TOL, what
    _exact(depth[~hit], r_depth[~hit].astype(np.float32), f"{what} far plane")


def _full_frame_vs_oracle(tree, cam, frame, o, d, opts=vv.RenderOptions(), what=""):
    rgb, alpha, depth, used = _camera_render(tree, cam, frame, opts)
    ref = oracle.render_rays(tree, o, d, frame, early_stop=opts.early_stop)
    _exact(used.reshape(-1), ref["used"], f"{what} sample counts")
    _check_images(rgb, alpha, depth, ref, what=what)
    return ref, (rgb, alpha, depth)


# ------------------------------------------------------------------ cfg2
@pytest.fixture(scope="module")
def cfg2():
    tree = synthetic.shell_tree()
    cam = synthetic.bench_camera()
    o, d = oracle.camera_rays(cam)
    return tree, cam, o, d


def test_cfg2_camera_kernel_full_frame(cuda, cfg2):
    """cfg2 production path (slice pass + sliced camera kernel, regular
    queue): all 2,073,600 pixels' sample counts bit-exact and images within
    1e-4 of the oracle, at two frames; the per-sample decode path too."""
    tree, cam, o, d = cfg2
    from paper_2202_06088_b200.device import replica

    assert replica(tree).dark_fraction < 0.5  # the regular-queue instantiation
    ref, _ = _full_frame_vs_oracle(tree, cam, 11, o, d, what="cfg2 f11")
    assert (ref["used"] > 0).mean() > 0.3
    _full_frame_vs_oracle(tree, cam, 29, o, d, what="cfg2 f29")
    _full_frame_vs_oracle(tree, cam, 3, o, d, vv.RenderOptions(frame_slice="per_sample"), what="cfg2 per-sample")


def test_cfg2_visits_bit_exact(cuda, cfg2):
    """Visited-leaf lists of the camera rays (render_ray_visits on the same
    fp64 rays) against the oracle's, on a 200k-pixel sample."""
    tree, cam, o, d = cfg2
    idx = np.sort(np.random.default_rng(5).choice(len(o), 200_000, replace=False))
    ref = oracle.render_rays(tree, o[idx], d[idx], 17, visits=True)
    used, start, leaf = vv.render_ray_visits(tree, o[idx], d[idx], 17)
    _exact(used, ref["used"], "counts")
    _exact(start, ref["visit_start"], "visit starts")
    _exact(leaf, ref["visit_leaf"], "visited leaves")


def test_camera_ray_agreement(cuda, cfg2):
    """Fraction of 1080p pixels whose GPU-order camera ray visits exactly the
    leaves the reference's Camera.rays ray (numpy BLAS) visits -- the
    reference's rays may differ in the last ulp.  Reported, and bounded."""
    tree, cam, o, d = cfg2
    ho, hd = cam.rays()  # the reference formula (render.py:74-83)
    diff = np.flatnonzero((hd != d).any(axis=1) | (ho != o).any(axis=1))
    agree = len(o)
    if len(diff):
        a = oracle.render_rays(tree, ho[diff], hd[diff], 11, visits=True)
        b = oracle.render_rays(tree, o[diff], d[diff], 11, visits=True)
        same = np.ones(len(diff), bool)
        for r in range(len(diff)):
            la = a["visit_leaf"][a["visit_start"][r]:a["visit_start"][r + 1]]
            lb = b["visit_leaf"][b["visit_start"][r]:b["visit_start"][r + 1]]
            same[r] = np.array_equal(la, lb)
        agree -= int((~same).sum())
    rate = agree / len(o)
    print(f"camera-ray visit agreement: {rate:.8f} ({len(diff)} of {len(o)} rays differ in some ulp)")
    assert rate >= 0.9999


# ------------------------------------------------------------------ cfg3
@pytest.fixture(scope="module")
def cfg3():
    tree = synthetic.motion_tree()
    cam = synthetic.bench_camera()
    o, d = oracle.camera_rays(cam)
    return tree, cam, o, d


def test_cfg3_long_queue_camera_kernel_full_frame(cuda, cfg3):
    """cfg3: the motion tree is ~90% dark, so render() runs the threshold-8
    long-queue sliced camera kernel -- full-frame counts bit-exact and images
    within 1e-4 of the oracle at four frames across the 60-frame sweep."""
    tree, cam, o, d = cfg3
    from paper_2202_06088_b200.device import replica

    assert replica(tree).dark_fraction > 0.5
    for f in (0, 15, 31, 45):
        ref, _ = _full_frame_vs_oracle(tree, cam, f, o, d, what=f"cfg3 f{f}")
        assert ref["shaded"].sum() > 0


def test_cfg3_per_sample_path(cuda, cfg3):
    tree, cam, o, d = cfg3
    _full_frame_vs_oracle(tree, cam, 20, o, d, vv.RenderOptions(frame_slice="per_sample"), what="cfg3 per-sample")


def test_cfg3_visits_bit_exact(cuda, cfg3):
    tree, cam, o, d = cfg3
    idx = np.sort(np.random.default_rng(6).choice(len(o), 100_000, replace=False))
    ref = oracle.render_rays(tree, o[idx], d[idx], 40, visits=True)
    used, start, leaf = vv.render_ray_visits(tree, o[idx], d[idx], 40)
    _exact(used, ref["used"], "counts")
    _exact(leaf, ref["visit_leaf"], "visited leaves")


@pytest.mark.parametrize("frames", [[8, 9, 10, 11], [50, 2, 33]])
def test_cfg3_shared_walk_playback_vs_oracle(cuda, cfg3, frames):
    """The threshold-8 shared-walk playback kernel (2..4 frames per walk):
    every frame bitwise equal to its single-frame render and within 1e-4 of
    the oracle on the full frame; render_sequence delivers the same bytes."""
    import torch

    tree, cam, o, d = cfg3
    h, w = cam.height, cam.width
    outs = [(torch.empty((h, w, 3), device=cuda), torch.empty((h, w), device=cuda), torch.empty((h, w), device=cuda))
            for _ in frames]
    vv.render_frames_into(tree, cam, frames, outs)
    torch.cuda.synchronize()
    seq = list(vv.render_sequence(tree, cam, frames))
    for f, (r, a, dd), s in zip(frames, outs, seq):
        rgb, alpha, depth, _ = _camera_render(tree, cam, f)
        _exact(r.cpu().numpy(), rgb, f"playback rgb {f}")
        _exact(a.cpu().numpy(), alpha, f"playback alpha {f}")
        _exact(dd.cpu().numpy(), depth, f"playback depth {f}")
        _exact(s.rgb, rgb, f"sequence rgb {f}")
        _exact(s.depth, depth, f"sequence depth {f}")
        ref = oracle.render_rays(tree, o, d, f)
        _check_images(r.cpu().numpy(), a.cpu().numpy(), dd.cpu().numpy(), ref, what=f"playback {f}")


# ------------------------------------------------------------------ cfg4
@pytest.fixture(scope="module")
def cfg4_small():
    g = load("cfg4_scene")
    trees = [synthetic.shell_tree(depth=8, n_max=2, frames=30, seed=i) for i in range(4)]
    scene, cam = synthetic.scene_config4(trees, 320, 180)
    cam_g = camera_from(g)
    assert np.array_equal(cam.c2w, cam_g.c2w) and (cam.width, cam.height) == (cam_g.width, cam_g.height)
    return g, scene, cam


@pytest.mark.parametrize("mode", ["auto", "per_sample", "per_frame"])
def test_cfg4_scene_vs_reference(cuda, cfg4_small, mode):
    """cfg4 shape (4 performers, S_3 = 0.8 non-rigid, shift|loop timemaps)
    against the reference's compose.render_scene: "auto" and "per_sample"
    decode per sample in the lean scene kernel (the one cfg4 runs at
    1080p), "per_frame" slices every performer (k_render_scene)."""
    g, scene, cam = cfg4_small
    opts = vv.RenderOptions(frame_slice=mode)
    for gf in (7, 22):
        _exact([i.local_frame(gf) for i in scene.instances], g[f"g{gf}_local_frames"], "local frames")
        img = vv.render_scene(scene, cam, gf, opts)
        assert np.abs(img - g[f"g{gf}_image"]).max() < TOL, (mode, gf)
        img2, blended, layers = vv.render_scene(scene, cam, gf, opts, want_layers=True)
        assert np.abs(img2 - g[f"g{gf}_image"]).max() < TOL
        assert np.abs(np.asarray(blended.alpha) - g[f"g{gf}_alpha"]).max() < TOL
        hit = g[f"g{gf}_alpha"] >= 1e-3
        assert np.abs(np.asarray(blended.depth)[hit] - g[f"g{gf}_depth"][hit]).max() < TOL


def test_cfg4_lean_kernel_selected(cuda, cfg4_small):
    """At the cfg4 shape every performer's footprint is small against its leaf
    count, so "auto" decodes per sample: the lean scene kernel."""
    import ctypes

    from paper_2202_06088_b200 import _native
    from paper_2202_06088_b200.compose import scene_instances

    g, scene, cam = cfg4_small
    descs, reps, _ = scene_instances(scene, cam, 7)
    modes = (ctypes.c_int32 * len(descs))()
    _native.check(_native.lib().vv_scene_decode_modes(descs, len(descs), None, ctypes.byref(cam.desc()), modes))
    assert list(modes) == [0, 0, 0, 0]


# ------------------------------------------------------------------ cfg5
def test_cfg5_stereo_eye_full_frame_and_shards(cuda):
    """cfg5: one 2160x2160 eye on the full frame against the oracle (counts
    bit-exact, images within 1e-4); the 8-shard direct tile render (64x64
    tiles interleaved, each shard writing only its pixels) bitwise equal to
    render() of that eye."""
    import ctypes

    import torch

    from paper_2202_06088_b200 import _native
    from paper_2202_06088_b200.device import replica, stream_ptr

    tree = synthetic.shell_tree()
    left, right = synthetic.stereo_cameras()
    o, d = oracle.camera_rays(right)
    rgb, alpha, depth = _full_frame_vs_oracle(tree, right, 9, o, d, what="cfg5 right eye")[1]
    rep = replica(tree, cuda)
    n = left.height * left.width
    planes = torch.full((5 * n,), float("nan"), device=cuda)
    ref = vv.render(tree, left, 9)
    oc, cd = vv.RenderOptions().c_struct(), left.desc()
    for s in range(8):
        _native.check(_native.lib().vv_render_camera_tiles_direct(
            rep.handle, 9, None, ctypes.byref(oc), ctypes.byref(cd), 64, s, 8, planes.data_ptr(),
            planes.data_ptr() + 12 * n, planes.data_ptr() + 16 * n, 0, stream_ptr(cuda)))
    torch.cuda.synchronize()
    p = planes.cpu().numpy()
    _exact(p[:3 * n].reshape(ref.rgb.shape), ref.rgb, "sharded rgb")
    _exact(p[3 * n:4 * n].reshape(ref.alpha.shape), ref.alpha, "sharded alpha")
    _exact(p[4 * n:].reshape(ref.depth.shape), ref.depth, "sharded depth")
