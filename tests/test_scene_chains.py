"""render_scene without host fallbacks: scenes the fused kernel cannot take
in one launch (more than 16 instances, mixed n_max) chain launches that carry
the per-pixel Algorithm-1 state (f64) on the device; want_layers renders the
per-instance layers with single-instance launches; any number of lights.
Checked against the reference's own layer-then-blend flow restated on the
host (render_instance layers + compose.blend_layers, compose.py:373-475)."""

import numpy as np
import pytest

import paper_2202_06088_b200 as vv
from paper_2202_06088_b200.compose import blend_layers, render_instance
from trees import random_payload_tree

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _tr(x, y, z):
    m = np.eye(4)
    m[:3, 3] = [x, y, z]
    return m


def _host_flow(scene, cam, g):
    layers = [render_instance(i, cam, g) for i in scene.visible_instances()]
    raw = blend_layers(layers)
    safe = np.maximum(raw.alpha, 1e-300)[..., None]
    rgb = np.where(raw.alpha[..., None] > 0.0, raw.rgb / safe, 0.0) if len(layers) > 1 else raw.rgb
    a = raw.alpha[..., None]
    return a * rgb + (1.0 - a) * scene.background, layers


def test_more_than_16_instances_chained(cuda):
    rng = np.random.default_rng(3)
    trees = [random_payload_tree(rng, depth=3, fill=0.5, frames=6, sigma_scale=5.0) for _ in range(3)]
    insts = []
    for i in range(21):
        a = _tr(0.45 * (i % 7) - 1.3, 0.35 * (i // 7), 0.1 * (i % 3))
        if i % 5 == 4:
            a = a @ np.diag([0.8, 0.8, 0.8, 1.0])  # some non-rigid
        insts.append(vv.SceneInstance(name=f"i{i}", tree=trees[i % 3], affine=a,
                                      timemap=vv.TimeMap.parse(f"shift({i % 4})")))
    scene = vv.Scene(instances=insts, background=np.array([0.2, 0.1, 0.3]))
    cam = vv.Camera.look_at([0.2, -4.0, 1.5], [0.2, 0.5, 0.4], width=48, height=32)
    for g in (0, 3):
        img = vv.render_scene(scene, cam, g)
        ref, _ = _host_flow(scene, cam, g)
        assert np.abs(img - ref).max() < TOL


def test_mixed_nmax_chained_and_layers(cuda):
    rng = np.random.default_rng(4)
    t1 = random_payload_tree(rng, depth=3, fill=0.5, frames=6, n_max=1, sigma_scale=6.0)
    t2 = random_payload_tree(rng, depth=3, fill=0.5, frames=6, n_max=2, sigma_scale=6.0)
    t3 = random_payload_tree(rng, depth=2, fill=0.7, frames=6, n_max=3, sigma_scale=4.0)
    insts = [vv.SceneInstance(name="a", tree=t1, affine=_tr(0.0, 0.0, 0.0)),
             vv.SceneInstance(name="b", tree=t2, affine=_tr(0.6, 0.4, 0.1), timemap=vv.TimeMap.parse("reverse")),
             vv.SceneInstance(name="c", tree=t2, affine=_tr(-0.7, 0.2, 0.0) @ np.diag([1.2, 1.2, 1.2, 1.0])),
             vv.SceneInstance(name="d", tree=t3, affine=_tr(0.1, 0.9, 0.2), yaw_rate=10.0),
             vv.SceneInstance(name="e", tree=t1, affine=_tr(0.3, -0.6, 0.3))]
    scene = vv.Scene(instances=insts, background=np.array([0.05, 0.1, 0.15]))
    cam = vv.Camera.look_at([0.3, -3.0, 1.6], [0.3, 0.5, 0.4], width=40, height=36)
    for g in (1, 4):
        img = vv.render_scene(scene, cam, g)
        ref, layers = _host_flow(scene, cam, g)
        assert np.abs(img - ref).max() < TOL
        img2, blended, lays = vv.render_scene(scene, cam, g, want_layers=True)
        assert np.abs(img2 - ref).max() < TOL
        for a, b in zip(lays, layers):
            assert np.abs(np.asarray(a.alpha) - b.alpha).max() < TOL
            assert np.abs(np.asarray(a.rgb) - b.rgb).max() < TOL
        raw = blend_layers(layers)
        assert np.abs(np.asarray(blended.alpha) - raw.alpha).max() < TOL


def test_many_lights(cuda):
    """More lights than the old 16-light cap: falloff-only lights, all applied."""
    rng = np.random.default_rng(5)
    t = random_payload_tree(rng, depth=3, fill=0.5, frames=4, sigma_scale=6.0)
    insts = [vv.SceneInstance(name="a", tree=t, affine=_tr(0.0, 0.0, 0.5))]
    lights = [vv.Light(position=(np.cos(k) * 2, np.sin(k) * 2, 2.0 + 0.05 * k), cast_shadows=False,
                       falloff_enabled=True, falloff_r0=2.0 + 0.1 * k, falloff_min_scale=0.5) for k in range(20)]
    scene = vv.Scene(instances=insts, lights=lights, background=np.array([0.3, 0.3, 0.3]))
    cam = vv.Camera.look_at([0.5, -2.5, 1.8], [0.5, 0.5, 0.8], width=32, height=24)
    img, blended, layers = vv.render_scene(scene, cam, 1, want_layers=True)
    from paper_2202_06088_b200.compose import falloff_pass

    base = render_instance(insts[0], cam, 1)
    rgb = base.rgb.copy()
    for l in lights:
        rgb = rgb * falloff_pass(vv.LayerImages(rgb, base.alpha, base.depth), cam, l)[..., None]
    a = base.alpha[..., None]
    ref = a * rgb + (1 - a) * scene.background
    assert np.abs(img - ref).max() < TOL
    assert np.abs(np.asarray(blended.rgb) - rgb).max() < TOL


@pytest.mark.parametrize("lit", [False, True])
def test_render_scene_sequence_bitwise(cuda, lit):
    """The compose loop (cli.py:184-200) pipelined: every yielded image is
    bitwise render_scene(scene, cam_i, g_i), with a camera per frame (the
    orbit) and with lights; closing the generator early is safe."""
    rng = np.random.default_rng(6)
    t = random_payload_tree(rng, depth=4, fill=0.4, frames=8, sigma_scale=6.0)
    insts = [vv.SceneInstance(name="a", tree=t, affine=_tr(0.0, 0.0, 0.3), timemap=vv.TimeMap.parse("shift(2)")),
             vv.SceneInstance(name="b", tree=t, affine=_tr(0.7, 0.3, 0.2) @ np.diag([0.9, 0.9, 0.9, 1.0]),
                              yaw_rate=12.0)]
    lights = [vv.Light(position=(0.9, 0.4, 3.5), blur_sigma=1.0, shadow_resolution=64, falloff_enabled=True)] if lit \
        else []
    scene = vv.Scene(instances=insts, lights=lights, background=np.array([0.1, 0.2, 0.3]))
    frames = list(range(7))
    cams = [vv.Camera.look_at([0.5 + 2.5 * np.cos(0.3 * i), 0.5 + 2.5 * np.sin(0.3 * i), 1.6], [0.5, 0.5, 0.5],
                              width=40, height=30) for i in frames]
    seq = list(vv.render_scene_sequence(scene, cams, frames))
    assert len(seq) == len(frames)
    for g, c, img in zip(frames, cams, seq):
        assert np.array_equal(img, vv.render_scene(scene, c, g)), g
    one = list(vv.render_scene_sequence(scene, cams[2], [5, 1]))
    assert np.array_equal(one[0], vv.render_scene(scene, cams[2], 5))
    assert np.array_equal(one[1], vv.render_scene(scene, cams[2], 1))
    gen = vv.render_scene_sequence(scene, cams, frames)
    first = next(gen)
    gen.close()
    assert np.array_equal(first, seq[0])
    with pytest.raises(ValueError):
        vv.render_scene_sequence(scene, cams[:3], frames)
