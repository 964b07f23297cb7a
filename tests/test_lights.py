"""Lighting passes (compose.py:539-619) against the reference: lit
render_scene images, shadow maps, background factors and falloff scales
(tests/golden/lights.npz), plus the reference's lighting tests
(test_compose.py:390-463)."""
import math

import numpy as np
import pytest

from golden_util import load, tree_from
import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import hh
from paper_2202_06088_b200.compose import (Light, Scene, SceneInstance, ShadowMap, TimeMap, falloff_pass,
                                           shadow_pass)
from paper_2202_06088_b200.render import LayerImages

TOL = 1e-4


def _tr(x, y, z):
    m = np.eye(4)
    m[:3, 3] = [x, y, z]
    return m


def _scene(g):
    ta, tb = tree_from(g, "ta_"), tree_from(g, "tb_")
    insts = [SceneInstance(name="a", tree=ta, affine=_tr(0.0, 0.0, 0.6)),
             SceneInstance(name="b", tree=tb, affine=_tr(1.3, 0.2, 0.4), timemap=TimeMap.parse("shift(1)"))]
    lights = [Light(position=(0.9, 0.4, 3.5), blur_sigma=1.5, shadow_resolution=96, falloff_enabled=True,
                    falloff_r0=2.5, falloff_min_scale=0.2),
              Light(position=(-0.5, 1.5, 2.0), cast_shadows=False, falloff_enabled=True, falloff_r0=1.5),
              Light(position=(2.0, -1.0, 2.5), blur_sigma=0.0, shadow_resolution=64, shadow_strength=0.5)]
    cam = vv.Camera.look_at([0.8, -3.0, 2.2], [0.8, 0.5, 0.3], width=28, height=22)
    assert np.array_equal(cam.c2w, g["cam_c2w"])
    return Scene(instances=insts, lights=lights, background=np.array([0.6, 0.65, 0.7])), cam


def _wall():
    h000 = 1.0 / (math.sqrt(2.0) * math.pi)
    k = hh.basis_count(1)
    rows = []
    coords = [(0, y, z) for y in range(2) for z in range(2)]
    for _ in coords:
        row = np.zeros(2 * 3 + 3 * k, dtype=np.float32)
        row[0] = 800.0
        for ch in range(3):
            row[6 + ch] = math.log(0.4 / 0.6) / h000
        rows.append(row)
    return vv.VOctree.from_cells(np.array(coords), np.stack(rows), vv.make_bump_bases(4, 3), 1, depth=1)


# ---------------------------------------------------------------- CPU
def test_light_validation():
    with pytest.raises(ValueError, match="off the ground plane"):
        Light(position=(0.0, 0.0, 0.0), ground_plane=(0, 0, 1, 0))
    with pytest.raises(ValueError, match="blur_sigma"):
        Light(position=(0, 0, 2), blur_sigma=-1.0)


def test_falloff_pass_vs_reference():
    g = load("lights")
    scene, cam = _scene(g)
    for fr in (0, 2):
        layer = LayerImages(rgb=g[f"g{fr}_blended_rgb"], alpha=g[f"g{fr}_blended_alpha"],
                            depth=g[f"g{fr}_blended_depth"])
        np.testing.assert_allclose(falloff_pass(layer, cam, scene.lights[1]), g[f"g{fr}_falloff1"], atol=1e-12)


def test_falloff_formula_and_monotonicity():
    """test_compose.py:441-463 of the reference."""
    rng = np.random.default_rng(51)
    light = Light(position=(0.0, 0.0, 0.0), ground_plane=(0, 0, 1, -5.0), falloff_r0=2.0, falloff_min_scale=0.05)
    h = w = 4
    cam = vv.Camera.look_at([0.0, 0.0, 0.0], [0.0, 1.0, 0.0], width=w, height=h)
    depths = rng.uniform(0.5, 6.0, (h, w))
    layer = LayerImages(rgb=np.full((h, w, 3), 0.5), alpha=np.ones((h, w)), depth=depths)
    scale = falloff_pass(layer, cam, light)
    np.testing.assert_allclose(scale, np.clip(4.0 / (4.0 + depths ** 2), 0.05, 1.0), atol=1e-9)
    layer0 = LayerImages(rgb=layer.rgb, alpha=layer.alpha, depth=np.zeros((h, w)))
    np.testing.assert_allclose(falloff_pass(layer0, cam, light), 1.0, atol=1e-12)
    layer_r0 = LayerImages(rgb=layer.rgb, alpha=layer.alpha, depth=np.full((h, w), 2.0))
    np.testing.assert_allclose(falloff_pass(layer_r0, cam, light), 0.5, atol=1e-12)
    flat = scale.ravel()[np.argsort(depths.ravel())]
    assert (np.diff(flat) <= 1e-12).all()


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_lit_render_scene_vs_reference(cuda):
    g = load("lights")
    scene, cam = _scene(g)
    for fr in (0, 2):
        img = vv.render_scene(scene, cam, fr)
        assert np.abs(img - g[f"g{fr}_image"]).max() < TOL
        host, _, _ = vv.render_scene(scene, cam, fr, want_layers=True)  # host lighting path
        assert np.abs(host - g[f"g{fr}_image"]).max() < TOL


@pytest.mark.gpu
def test_shadow_maps_vs_reference(cuda):
    g = load("lights")
    scene, cam = _scene(g)
    for fr in (0, 2):
        sm = shadow_pass(scene.instances, scene.lights[0], fr)
        assert np.array_equal(sm.cam.c2w, g[f"g{fr}_shadow0_c2w"])
        assert np.abs(sm.alpha - g[f"g{fr}_shadow0"]).max() < 1e-5
        assert np.abs(sm.background_factor(cam) - g[f"g{fr}_bgfac0"]).max() < 1e-5
        sm2 = shadow_pass(scene.instances, scene.lights[2], fr)  # blur_sigma 0: no blur
        assert np.abs(sm2.alpha - g[f"g{fr}_shadow2"]).max() < 1e-5


@pytest.mark.gpu
def test_shadow_blur_matches_scipy(cuda):
    from scipy.ndimage import gaussian_filter

    g = load("lights")
    scene, _ = _scene(g)
    light = Light(position=(0.9, 0.4, 3.5), blur_sigma=2.3, shadow_resolution=80)
    sharp = shadow_pass(scene.instances, Light(position=(0.9, 0.4, 3.5), blur_sigma=0.0, shadow_resolution=80), 0)
    blurred = shadow_pass(scene.instances, light, 0)
    ref = gaussian_filter(sharp.alpha, 2.3, mode="constant", cval=0.0)
    assert np.abs(blurred.alpha - ref).max() < 1e-12


@pytest.mark.gpu
def test_shadow_no_instances_no_darkening(cuda):
    sm = shadow_pass([], Light(position=(0.5, 0.5, 3.0)))
    pts = np.random.default_rng(50).uniform(-1, 2, size=(50, 3))
    pts[:, 2] = 0.0
    np.testing.assert_allclose(sm.factor_at_points(pts), 1.0, atol=1e-12)


@pytest.mark.gpu
def test_shadow_centroid_under_opaque_cube(cuda):
    inst = SceneInstance(name="c", tree=_wall(), affine=_tr(0.6, 0.2, 0.8))
    light = Light(position=(0.85, 0.7, 4.0), ground_plane=(0, 0, 1, 0), blur_sigma=0.0, shadow_resolution=160)
    sm = shadow_pass([inst], light)
    xs = np.linspace(-0.5, 2.2, 220)
    ys = np.linspace(-0.5, 2.0, 200)
    gx, gy = np.meshgrid(xs, ys, indexing="ij")
    pts = np.stack([gx.ravel(), gy.ravel(), np.zeros(gx.size)], 1)
    dark = 1.0 - sm.factor_at_points(pts)
    m = dark.sum()
    texel = 4.0 / (0.7 * 160)
    assert abs(float((pts[:, 0] * dark).sum() / m) - 0.85) < texel
    assert abs(float((pts[:, 1] * dark).sum() / m) - 0.7) < texel


@pytest.mark.gpu
def test_shadow_blur_preserves_mass(cuda):
    inst = SceneInstance(name="c", tree=_wall(), affine=_tr(0.6, 0.2, 0.8))
    base = dict(position=(0.85, 0.7, 4.0), ground_plane=(0, 0, 1, 0), shadow_resolution=160)
    m0 = shadow_pass([inst], Light(blur_sigma=0.0, **base)).alpha.sum()
    m1 = shadow_pass([inst], Light(blur_sigma=2.0, **base)).alpha.sum()
    assert abs(m1 - m0) / m0 < 0.02
