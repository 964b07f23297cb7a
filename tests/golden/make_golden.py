"""Generate tests/golden/*.npz from the REFERENCE implementation.

Run in a container that has the reference checked out at /root/reference
(it is not present on GPU boxes; the committed .npz files travel instead):

    python tests/golden/make_golden.py

Every case stores its inputs (tree arrays or the generator arguments, rays,
frame, options) and the reference outputs:

* render_rays premult/alpha/tbar (render.py:182-215, kernels.py:410-652);
* per-ray ``used`` counts and visited leaf rows from Trainer._forward
  (train.py:269-296; shade_forward_kernel, kernels.py:655-743) -- the
  sample-count oracle named in SURVEY.md section 8(c);
* full segment lists from count/collect_segments_kernel (kernels.py:313-367);
* build_frame_cache sigma/q (kernels.py:397-407);
* LayerImages from render() and images from compose.render_scene;
* .voct bytes from VOctree.to_bytes;
* compose.paint results (edit channels, skipped pixels) and the per-ray
  termination leaves of its loop (compose.py:508-522).

    python tests/golden/make_golden.py [case ...]   # default: every case
"""

from __future__ import annotations

import hashlib
import math
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vv_numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

from voxvid import hh as rhh  # noqa: E402
from voxvid import kernels as rk  # noqa: E402
from voxvid import temporal as rt  # noqa: E402
from voxvid.compose import (  # noqa: E402
    Light,
    Scene,
    SceneInstance,
    TimeMap,
    falloff_pass,
    paint,
    render_scene,
    shadow_pass,
)
from voxvid.octree import VOctree  # noqa: E402
from voxvid.render import Camera, RenderOptions, build_frame_cache, render, render_rays  # noqa: E402
from voxvid.train import TrainConfig, Trainer  # noqa: E402


def tree_arrays(tree, prefix="tree_"):
    out = {
        prefix + "depth": np.int64(tree.depth),
        prefix + "n_max": np.int64(tree.n_max),
        prefix + "node_child": tree.node_child,
        prefix + "leaf_coords": tree.leaf_coords,
        prefix + "leaf_data": tree.leaf_data,
        prefix + "a": tree.bases.a,
        prefix + "b": tree.bases.b,
        prefix + "bbox_lo": tree.bbox_lo,
        prefix + "side": np.float64(tree.side),
    }
    if tree.has_edits:
        out[prefix + "edit_rgb"] = tree.edit_rgb
        out[prefix + "edit_t"] = tree.edit_t
    return out


def random_payload_tree(rng, depth=2, fill=0.6, frames=4, coeff_count=3, n_max=2, sigma_scale=2.0):
    # tests/util.py:41-53 of the reference
    res = 1 << depth
    occ = rng.random((res, res, res)) < fill
    coords = np.argwhere(occ)
    k = rhh.basis_count(n_max)
    data = rng.normal(scale=0.5, size=(len(coords), 2 * coeff_count + 3 * k))
    data[:, 0] = rng.uniform(0.2, sigma_scale, size=len(coords))
    return VOctree.from_cells(coords, data.astype(np.float32), rt.make_bump_bases(frames, coeff_count), n_max,
                              depth=depth)


def forward_used(tree, origins, dirs, frame, early_stop):
    tr = Trainer(tree, TrainConfig(early_stop=early_stop, coeff_count=tree.coeff_count, n_max=tree.n_max))
    premult, alpha, tbar, aux = tr._forward(origins, dirs, np.full(len(origins), frame, dtype=np.int64))
    used = aux["used"]
    starts = aux["start"]
    vs = np.zeros(len(origins) + 1, np.int64)
    vs[1:] = np.cumsum(used)
    vl = np.concatenate([aux["seg_leaf"][starts[r]: starts[r] + used[r]] for r in range(len(origins))]) \
        if len(origins) else np.zeros(0, np.int64)
    return dict(fwd_premult=premult, fwd_alpha=alpha, fwd_tbar=tbar, used=used.astype(np.int32),
                visit_start=vs, visit_leaf=vl.astype(np.int64))


def segments(tree, origins, dirs, tmin=0.0, tmax=1e30):
    n = len(origins)
    cnt = np.empty(n, np.int64)
    rk.count_segments_kernel(tree.node_child, tree.depth, tree.bbox_lo, tree.side, origins, dirs, tmin, tmax, cnt)
    start = np.zeros(n + 1, np.int64)
    start[1:] = np.cumsum(cnt)
    tot = int(start[-1])
    leaf = np.empty(tot, np.int64)
    t0 = np.empty(tot)
    t1 = np.empty(tot)
    rk.collect_segments_kernel(tree.node_child, tree.depth, tree.bbox_lo, tree.side, origins, dirs, tmin, tmax,
                               start[:-1].copy(), leaf, t0, t1)
    return dict(seg_start=start, seg_leaf=leaf, seg_t0=t0, seg_t1=t1)


def render_case(tree, origins, dirs, frame, early_stop, with_used=True, cache=None):
    opts = RenderOptions(early_stop=early_stop)
    p, a, t = render_rays(tree, origins, dirs, frame, opts, cache=cache)
    out = dict(premult=p, alpha=a, tbar=t)
    if with_used:
        out.update(forward_used(tree, origins, dirs, frame, early_stop))
    return out


def edge_rays(rng, n_random=1500):
    """Random rays plus the traversal's edge cases: axis-aligned and
    zero-component directions, origins on grid planes and inside the cube,
    rays aimed exactly at grid corners and edges."""
    o, d = [], []
    for _ in range(n_random):
        oo = rng.uniform(-0.5, 1.5, 3) if rng.random() < 0.6 else rng.uniform(0.0, 1.0, 3)
        dd = rng.normal(size=3)
        if rng.random() < 0.2:
            dd[rng.integers(3)] = 0.0
        if rng.random() < 0.1:
            dd[rng.integers(3)] = 0.0
        if np.linalg.norm(dd) == 0:
            dd = np.array([1.0, 0.0, 0.0])
        o.append(oo)
        d.append(dd / np.linalg.norm(dd))
    grid = np.arange(0, 17) / 16.0
    for _ in range(300):  # origins on planes, axis directions
        oo = rng.choice(grid, 3)
        ax = rng.integers(3)
        dd = np.zeros(3)
        dd[ax] = rng.choice([-1.0, 1.0])
        oo[ax] = -0.25 if dd[ax] > 0 else 1.25
        o.append(oo)
        d.append(dd)
    for _ in range(300):  # aimed at lattice corners/edges from outside
        tgt = rng.choice(grid, 3)
        src = tgt + rng.choice([-1.0, 1.0], 3) * rng.choice([0.5, 1.0, 2.0], 3)
        dd = tgt - src
        o.append(src)
        d.append(dd / np.linalg.norm(dd))
    for _ in range(100):  # exact diagonals through corners
        src = np.array([-0.5, -0.5, -0.5]) + rng.choice(grid[:4], 3) * 0.0
        dd = np.array([1.0, 1.0, 1.0]) * rng.choice([-1.0, 1.0], 3)
        src = np.where(dd > 0, -0.5, 1.5) + rng.choice(grid, 3) * 0.0
        o.append(src)
        d.append(dd / np.linalg.norm(dd))
    return np.ascontiguousarray(o, dtype=np.float64), np.ascontiguousarray(d, dtype=np.float64)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def cfg4_scene_case():
    """BASELINE configs[3] shape at reduced size: the SURVEY 8(d) cfg4 scene
    (4 shell performers, affines T(1.1(i-1.5),0,0) T(c) Rz(0.5 i) S_i T(-c)
    with S_3 = 0.8 I -- the non-rigid per-ray pull-back --, timemaps
    shift(3i)|loop(30)) through the reference's compose.render_scene, with
    depth-8 trees (seeds 0-3) at 320x180, global frames 7 and 22."""
    from paper_2202_06088_b200 import synthetic

    trees = []
    for i in range(4):
        t = synthetic.shell_tree(depth=8, n_max=2, frames=30, seed=i)
        rt_ = VOctree.from_cells(t.leaf_coords, t.leaf_data, rt.TemporalBases(t.bases.a, t.bases.b), 2, depth=8)
        assert np.array_equal(rt_.node_child, t.node_child)
        trees.append(rt_)
    scene_ours, cam_ours = synthetic.scene_config4(trees, 320, 180)
    insts = [SceneInstance(name=i.name, tree=i.tree, affine=i.affine, timemap=TimeMap.parse(str(i.timemap)))
             for i in scene_ours.instances]
    scene = Scene(instances=insts)
    cam = Camera(cam_ours.width, cam_ours.height, cam_ours.fx, cam_ours.fy, cam_ours.cx, cam_ours.cy, cam_ours.c2w)
    c = dict(cam_c2w=cam.c2w, cam_wh=np.array([cam.width, cam.height]),
             cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy]))
    for g in (7, 22):
        img, blended, layers = render_scene(scene, cam, g, want_layers=True)
        c[f"g{g}_image"] = img.astype(np.float32)
        c[f"g{g}_alpha"] = blended.alpha.astype(np.float32)
        c[f"g{g}_depth"] = blended.depth.astype(np.float32)
        c[f"g{g}_local_frames"] = np.array([i.local_frame(g) for i in insts])
        c[f"g{g}_layer_alpha_max"] = np.array([float(l.alpha.max()) for l in layers])
    return c


def joint_case():
    """Per-sample depth-ordered joint composition: the reference's own
    joint_segments_oracle (pkg/tests/util.py:205-245) -- every instance's
    leaf segments merged by world depth and composited once, no early stop
    -- on depth-separated instances (where SPEC.md:555 makes Alg. 1 equal to
    it) and on interleaved ones (where only the joint oracle is the truth)."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    from util import joint_segments_oracle

    rng = np.random.default_rng(91)
    ta = random_payload_tree(rng, depth=3, fill=0.5, frames=6, sigma_scale=6.0)
    tb = random_payload_tree(rng, depth=4, fill=0.3, frames=6, sigma_scale=9.0)

    def tr(x, y, z):
        m = np.eye(4)
        m[:3, 3] = [x, y, z]
        return m

    scl = np.diag([0.7, 0.7, 0.7, 1.0]) @ tr(0.2, 0.3, 0.1)
    bg = np.array([0.1, 0.12, 0.2])
    c = dict(tree_arrays(ta, "ta_"), **tree_arrays(tb, "tb_"), bg=bg)
    layouts = {
        # separated along the view direction: b entirely behind a for every ray
        "sep": [SceneInstance(name="a", tree=ta, affine=tr(0.0, 0.0, 0.0)),
                SceneInstance(name="b", tree=tb, affine=tr(0.0, 2.5, 0.0), timemap=TimeMap.parse("shift(2)"))],
        # interleaved: overlapping volumes, a scaled (non-rigid) one and a yaw
        "mix": [SceneInstance(name="a", tree=ta, affine=tr(0.0, 0.0, 0.0)),
                SceneInstance(name="b", tree=tb, affine=tr(0.25, 0.1, 0.05), timemap=TimeMap.parse("reverse")),
                SceneInstance(name="c", tree=ta, affine=scl, yaw_rate=20.0)],
    }
    cam = Camera.look_at([0.5, -2.2, 0.9], [0.5, 0.8, 0.5], width=24, height=20)
    c.update(cam_c2w=cam.c2w, cam_wh=np.array([cam.width, cam.height]),
             cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy]))
    for name, insts in layouts.items():
        for g in (0, 3):
            c[f"{name}_g{g}_joint"] = joint_segments_oracle(insts, cam, g, bg)
            c[f"{name}_g{g}_alg1"] = render_scene(Scene(instances=insts, background=bg), cam, g,
                                                  RenderOptions(early_stop=0.0))
    return c


EXTRA = {"cfg4_scene": cfg4_scene_case, "joint": joint_case}


def main():
    want = set(sys.argv[1:])
    cases = {}
    if want and want <= set(EXTRA):
        for name in sorted(want):
            path = HERE / f"{name}.npz"
            np.savez_compressed(path, **EXTRA[name]())
            print(f"{path.name}: {path.stat().st_size / 1024:.0f} KiB")
        return

    # A. scalar-reference case (test_render.py:103-113 shape)
    rng = np.random.default_rng(23)
    tree = random_payload_tree(rng, depth=2, fill=0.7)
    cam = Camera.look_at([2.0, 1.7, -0.6], [0.5, 0.5, 0.5], width=6, height=6)
    o, d = cam.rays()
    c = dict(tree_arrays(tree), origins=o, dirs=d, frame=np.int64(3))
    for tag, es in (("nostop", 0.0), ("stop", 1e-4)):
        for k, v in render_case(tree, o, d, 3, es).items():
            c[f"{tag}_{k}"] = v
    c.update(segments(tree, o, d))
    cases["scalar_d2"] = c

    # B. cache / multi-frame case (test_render.py:116-126 shape) incl. slice rows
    rng = np.random.default_rng(24)
    tree = random_payload_tree(rng, depth=3, fill=0.4)
    cam = Camera.look_at([-1.0, 2.0, 1.2], [0.5, 0.5, 0.5], width=24, height=24)
    o, d = cam.rays()
    c = dict(tree_arrays(tree), origins=o, dirs=d)
    for fr in (0, 2):
        for k, v in render_case(tree, o, d, fr, 1e-4).items():
            c[f"f{fr}_{k}"] = v
        cache = build_frame_cache(tree, fr)
        c[f"f{fr}_slice_sigma"] = cache.sigma
        c[f"f{fr}_slice_q"] = cache.q
        layer = render(tree, cam, fr)
        c[f"f{fr}_rgb"] = layer.rgb
        c[f"f{fr}_alpha_img"] = layer.alpha
        c[f"f{fr}_depth"] = layer.depth
    c["cam_c2w"] = cam.c2w
    c["cam_wh"] = np.array([cam.width, cam.height])
    c["cam_f"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy])
    cases["cache_d3"] = c

    # C. traversal edge cases, depth 4, n_max 1, sigma large enough to stop early
    rng = np.random.default_rng(5)
    tree = random_payload_tree(rng, depth=4, fill=0.35, n_max=1, sigma_scale=40.0)
    o, d = edge_rays(np.random.default_rng(55))
    c = dict(tree_arrays(tree), origins=o, dirs=d)
    c.update(segments(tree, o, d))
    for tag, es in (("nostop", 0.0), ("stop", 1e-4)):
        for k, v in render_case(tree, o, d, 1, es).items():
            c[f"{tag}_{k}"] = v
    # clipped t-range (ray_segments t_range)
    seg = segments(tree, o, d, tmin=0.3, tmax=1.7)
    for k, v in seg.items():
        c["clip_" + k] = v
    cases["edge_d4"] = c

    # D. config 1 (BASELINE.json configs[0]): depth 7 shell, n_max 1, T 16, 64x64, frame 5
    from paper_2202_06088_b200 import synthetic

    t1 = synthetic.shell_tree(depth=7, n_max=1, frames=16, seed=0)
    tree = VOctree.from_cells(t1.leaf_coords, t1.leaf_data, rt.TemporalBases(t1.bases.a, t1.bases.b), 1, depth=7)
    assert np.array_equal(tree.node_child, t1.node_child)
    cam = synthetic.bench_camera(64, 64)
    o, d = cam.rays()
    c = dict(origins=o, dirs=d, frame=np.int64(5), tree_sha=np.array(sha(t1.node_child, t1.leaf_data,
                                                                          t1.bases.a, t1.bases.b)))
    for k, v in render_case(tree, o, d, 5, 1e-4).items():
        c[k] = v
    layer = render(tree, cam, 5)
    c["rgb"], c["alpha_img"], c["depth"] = layer.rgb, layer.alpha, layer.depth
    c["cam_c2w"] = cam.c2w
    c.update(segments(tree, o, d))
    cases["cfg1"] = c

    # E. edits (kernels.py:547-555, 584-587)
    rng = np.random.default_rng(31)
    tree = random_payload_tree(rng, depth=3, fill=0.5, frames=6)
    tree.ensure_edit_arrays()
    sel = rng.choice(tree.n_leaves, size=tree.n_leaves // 3, replace=False)
    for i, row in enumerate(sel):
        tree.edit_rgb[row, :3] = rng.uniform(0.0, 1.0, 3)
        tree.edit_rgb[row, 3] = -1.0 if i % 3 else rng.uniform(0.0, 5.0)
        if i % 5 == 0:
            tree.edit_rgb[row, 3] = 0.0
        tree.edit_t[row] = (1, 4) if i % 2 else (0, 5)
    cam = Camera.look_at([2.1, -0.7, 1.5], [0.5, 0.5, 0.5], width=20, height=20)
    o, d = cam.rays()
    c = dict(tree_arrays(tree), origins=o, dirs=d)
    for fr in (0, 2):
        for ew in (1.0, 0.4):
            p, a, t = render_rays(tree, o, d, fr, RenderOptions(edit_weight=ew))
            c[f"f{fr}_w{int(ew * 10)}_premult"], c[f"f{fr}_w{int(ew * 10)}_alpha"], c[f"f{fr}_w{int(ew * 10)}_tbar"] = p, a, t
    cases["edits_d3"] = c

    # F. other truncations
    for n_max in (0, 3):
        rng = np.random.default_rng(40 + n_max)
        tree = random_payload_tree(rng, depth=3, fill=0.5, n_max=n_max, coeff_count=5, frames=5)
        cam = Camera.look_at([2.3, 1.1, -0.4], [0.5, 0.5, 0.5], width=12, height=12)
        o, d = cam.rays()
        c = dict(tree_arrays(tree), origins=o, dirs=d, frame=np.int64(2))
        for k, v in render_case(tree, o, d, 2, 1e-4).items():
            c[k] = v
        cases[f"nmax{n_max}"] = c

    # G. scene composition (compose.py:418-475): rigid, translated, scaled, yawing, timemapped
    rng = np.random.default_rng(48)
    tree_a = random_payload_tree(rng, depth=3, fill=0.5, frames=6, sigma_scale=8.0)
    tree_b = random_payload_tree(rng, depth=2, fill=0.7, frames=6, sigma_scale=6.0)

    def tr(x, y, z):
        m = np.eye(4)
        m[:3, 3] = [x, y, z]
        return m

    scale = np.diag([1.3, 1.3, 1.3, 1.0]) @ tr(-0.3, 0.1, 0.0)
    insts = [
        SceneInstance(name="a", tree=tree_a, affine=tr(0.0, 0.0, 0.0)),
        SceneInstance(name="b", tree=tree_b, affine=tr(1.2, 0.3, 0.0), timemap=TimeMap.parse("shift(2)")),
        SceneInstance(name="c", tree=tree_a, affine=scale, timemap=TimeMap.parse("reverse")),
        SceneInstance(name="d", tree=tree_b, affine=tr(-1.1, 0.4, 0.2), yaw_rate=15.0),
    ]
    scene = Scene(instances=insts, background=np.array([0.1, 0.12, 0.2]))
    cam = Camera.look_at([0.6, 4.0, 1.5], [0.5, 0.5, 0.4], width=20, height=16)
    c = dict(tree_arrays(tree_a, "ta_"), **tree_arrays(tree_b, "tb_"), cam_c2w=cam.c2w,
             cam_wh=np.array([cam.width, cam.height]), cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy]))
    for g in (0, 3):
        img, blended, layers = render_scene(scene, cam, g, want_layers=True)
        c[f"g{g}_image"] = img
        c[f"g{g}_alpha"] = blended.alpha
        c[f"g{g}_depth"] = blended.depth
        for i, l in enumerate(layers):
            c[f"g{g}_layer{i}_rgb"] = l.rgb
            c[f"g{g}_layer{i}_alpha"] = l.alpha
            c[f"g{g}_layer{i}_depth"] = l.depth
    single = Scene(instances=[insts[2]], background=np.array([0.1, 0.12, 0.2]))
    c["single_image"] = render_scene(single, cam, 1)
    cases["scene"] = c

    # H. .voct bytes (octree.py:371-411), with and without edits
    rng = np.random.default_rng(61)
    tree = random_payload_tree(rng, depth=3, fill=0.3, n_max=1)
    c = dict(tree_arrays(tree), voct=np.frombuffer(tree.to_bytes(), dtype=np.uint8))
    tree.ensure_edit_arrays()
    tree.edit_rgb[::3, :3] = 0.25
    tree.edit_t[::3] = (2, 3)
    c["voct_edits"] = np.frombuffer(tree.to_bytes(), dtype=np.uint8)
    c["edit_rgb"] = tree.edit_rgb
    c["edit_t"] = tree.edit_t
    cases["voct"] = c

    # I. basis tables (kernels.py:56-76)
    c = {}
    for n_max in range(4):
        tab = rk.basis_tables(n_max)
        for f in ("pair_n", "pair_l", "pair_norm", "k2pair", "k2sh", "sh_pref"):
            c[f"n{n_max}_{f}"] = getattr(tab, f)
    cases["tables"] = c

    # J. paint (compose.py:482-532)
    rng = np.random.default_rng(71)
    tree = random_payload_tree(rng, depth=4, fill=0.3, frames=6, n_max=1, sigma_scale=12.0)
    cam = Camera.look_at([2.2, -0.8, 1.4], [0.5, 0.5, 0.5], width=24, height=20)
    c = dict(tree_arrays(tree), cam_c2w=cam.c2w, cam_wh=np.array([cam.width, cam.height]),
             cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy]))
    # per-ray termination leaves at frame 1, threshold 0.9: the loop of
    # compose.py:508-522 over the reference's own ray_segments and sigma
    o, d = cam.rays()
    sig = np.maximum(0.0, tree.leaf_data[:, :tree.coeff_count].astype(np.float64)
                     @ tree.bases.a[1].astype(np.float64))
    term = np.full(len(o), -1, np.int64)
    for r in range(len(o)):
        acc, trans = 0.0, 1.0
        for seg in tree.ray_segments(o[r], d[r]):
            a = 1.0 - math.exp(-sig[seg.leaf] * seg.delta)
            acc += trans * a
            trans *= 1.0 - a
            if acc >= 0.9:
                term[r] = seg.leaf
                break
    c.update(origins=o, dirs=d, term_leaf=term)
    mask = rng.random((cam.height, cam.width)) < 0.5
    res = paint(tree, cam, mask, (0.9, 0.2, 0.1), (1, 4), alpha_threshold=0.9)
    c.update(p1_mask=mask, p1_edited=np.int64(res["edited_voxels"]),
             p1_skipped=np.array(res["skipped_pixels"], np.int64).reshape(-1, 2),
             p1_edit_rgb=tree.edit_rgb.copy(), p1_edit_t=tree.edit_t.copy())
    pix = np.array([[3, 4], [10, 2], [23, 19], [0, 0], [12, 10], [15, 9]])
    res = paint(tree, cam, pix, (0.1, 0.8, 0.3), (2, 5), alpha_threshold=0.5, target_density=7.5, frame=3)
    c.update(p2_pixels=pix, p2_edited=np.int64(res["edited_voxels"]),
             p2_skipped=np.array(res["skipped_pixels"], np.int64).reshape(-1, 2),
             p2_edit_rgb=tree.edit_rgb.copy(), p2_edit_t=tree.edit_t.copy())
    cases["paint"] = c

    # K. lighting passes (compose.py:539-619): shadow maps, falloff, lit render_scene
    rng = np.random.default_rng(81)
    tree_a = random_payload_tree(rng, depth=3, fill=0.5, frames=6, sigma_scale=8.0)
    tree_b = random_payload_tree(rng, depth=2, fill=0.7, frames=6, sigma_scale=6.0)

    def tr(x, y, z):
        m = np.eye(4)
        m[:3, 3] = [x, y, z]
        return m

    insts = [SceneInstance(name="a", tree=tree_a, affine=tr(0.0, 0.0, 0.6)),
             SceneInstance(name="b", tree=tree_b, affine=tr(1.3, 0.2, 0.4), timemap=TimeMap.parse("shift(1)"))]
    lights = [Light(position=(0.9, 0.4, 3.5), blur_sigma=1.5, shadow_resolution=96, falloff_enabled=True,
                    falloff_r0=2.5, falloff_min_scale=0.2),
              Light(position=(-0.5, 1.5, 2.0), cast_shadows=False, falloff_enabled=True, falloff_r0=1.5),
              Light(position=(2.0, -1.0, 2.5), blur_sigma=0.0, shadow_resolution=64, shadow_strength=0.5)]
    scene = Scene(instances=insts, lights=lights, background=np.array([0.6, 0.65, 0.7]))
    cam = Camera.look_at([0.8, -3.0, 2.2], [0.8, 0.5, 0.3], width=28, height=22)
    c = dict(tree_arrays(tree_a, "ta_"), **tree_arrays(tree_b, "tb_"), cam_c2w=cam.c2w,
             cam_wh=np.array([cam.width, cam.height]), cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy]))
    for g in (0, 2):
        img, blended, _ = render_scene(scene, cam, g, want_layers=True)
        c[f"g{g}_image"] = img
        c[f"g{g}_blended_rgb"] = blended.rgb
        c[f"g{g}_blended_alpha"] = blended.alpha
        c[f"g{g}_blended_depth"] = blended.depth
        sm = shadow_pass(insts, lights[0], g)
        c[f"g{g}_shadow0"] = sm.alpha
        c[f"g{g}_shadow0_c2w"] = sm.cam.c2w
        c[f"g{g}_bgfac0"] = sm.background_factor(cam)
        sm2 = shadow_pass(insts, lights[2], g)
        c[f"g{g}_shadow2"] = sm2.alpha
        c[f"g{g}_falloff1"] = falloff_pass(blended, cam, lights[1])
    cases["lights"] = c

    for name, fn in EXTRA.items():
        if not want or name in want:
            cases[name] = fn()
    for name, arrays in cases.items():
        if want and name not in want:
            continue
        path = HERE / f"{name}.npz"
        np.savez_compressed(path, **arrays)
        print(f"{path.name}: {path.stat().st_size / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
