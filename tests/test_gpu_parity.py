"""GPU parity tests: the CUDA path (through the C ABI) against the reference's
golden vectors and the CPU oracle.

Contract (BASELINE.json north_star): visited-leaf indices and per-ray sample
counts bit-exact; RGB/alpha/depth within 1e-4 absolute.  Segment lists
(leaf, t_in, t_out) are bit-exact as well.  alpha/tbar are float64 with the
reference's operation order; they are compared at 1e-12 (CUDA exp() may
differ from glibc by 1 ulp).
"""

import numpy as np
import pytest

from golden_util import camera_from, load, tree_from
from oracle import oracle
import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import synthetic

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _exact(a, b, what=""):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    assert np.array_equal(a, b), f"{what}: {np.count_nonzero(a != b)} mismatches"


def _check_rays(tree, o, d, frame, g, prefix="", early_stop=1e-4):
    opts = vv.RenderOptions(early_stop=early_stop)
    p, a, t, st = vv.render_rays(tree, o, d, frame, opts, stats=True)
    assert np.abs(a - g[prefix + "alpha"]).max() <= 1e-12
    assert np.abs(t - g[prefix + "tbar"]).max() <= 1e-9
    assert np.abs(p - g[prefix + "premult"]).max() <= TOL
    if prefix + "used" in g:
        _exact(st["sample_count"], g[prefix + "used"], "sample counts")
        used, start, leaf = vv.render_ray_visits(tree, o, d, frame, opts)
        _exact(used, g[prefix + "used"], "visit counts")
        _exact(start, g[prefix + "visit_start"], "visit starts")
        _exact(leaf, g[prefix + "visit_leaf"], "visited leaves")
    return p, a, t, st


@pytest.mark.parametrize("tag,es", [("nostop", 0.0), ("stop", 1e-4)])
def test_scalar_case(cuda, tag, es):
    g = load("scalar_d2")
    _check_rays(tree_from(g), g["origins"], g["dirs"], int(g["frame"]), g, f"{tag}_", es)


@pytest.mark.parametrize("tag,es", [("nostop", 0.0), ("stop", 1e-4)])
def test_edge_rays(cuda, tag, es):
    g = load("edge_d4")
    _check_rays(tree_from(g), g["origins"], g["dirs"], 1, g, f"{tag}_", es)


@pytest.mark.parametrize("clip", [False, True])
def test_segments_bit_exact(cuda, clip):
    g = load("edge_d4")
    tree = tree_from(g)
    args = (0.3, 1.7) if clip else (0.0, 1e30)
    start, leaf, t0, t1 = vv.collect_segments(tree, g["origins"], g["dirs"], *args)
    p = "clip_" if clip else ""
    _exact(start, g[p + "seg_start"], "starts")
    _exact(leaf, g[p + "seg_leaf"], "leaves")
    _exact(t0, g[p + "seg_t0"], "t0")
    _exact(t1, g[p + "seg_t1"], "t1")
    cnt = vv.count_segments(tree, g["origins"], g["dirs"], *args)
    _exact(cnt, np.diff(g[p + "seg_start"]), "counts")


def test_ray_segments_api(cuda):
    g = load("scalar_d2")
    tree = tree_from(g)
    o, d = g["origins"], g["dirs"]
    for r in range(len(o)):
        segs = tree.ray_segments(o[r], d[r])
        s0, s1 = g["seg_start"][r], g["seg_start"][r + 1]
        assert [s.leaf for s in segs] == list(g["seg_leaf"][s0:s1])
        assert [s.t_enter for s in segs] == list(g["seg_t0"][s0:s1])


@pytest.mark.parametrize("frame", [0, 2])
def test_cache_bitwise_and_slice(cuda, frame):
    g = load("cache_d3")
    tree = tree_from(g)
    o, d = g["origins"], g["dirs"]
    p, a, t, st = _check_rays(tree, o, d, frame, g, f"f{frame}_")
    cache = vv.build_frame_cache(tree, frame)
    pc, ac, tc, stc = vv.render_rays(tree, o, d, frame, cache=cache, stats=True)
    _exact(pc, p, "cached premult")
    _exact(ac, a, "cached alpha")
    _exact(tc, t, "cached tbar")
    _exact(stc["sample_count"], st["sample_count"], "cached counts")
    _exact(cache.sigma.cpu().numpy(), g[f"f{frame}_slice_sigma"], "slice sigma")
    assert np.abs(cache.q.cpu().numpy() - g[f"f{frame}_slice_q"]).max() < 1e-5
    cam = camera_from(g)
    plain = vv.render(tree, cam, frame)
    cached = vv.render(tree, cam, frame, cache=cache)
    for x, y in zip((plain.rgb, plain.alpha, plain.depth), (cached.rgb, cached.alpha, cached.depth)):
        _exact(x, y, "cached image")
    assert np.abs(plain.rgb - g[f"f{frame}_rgb"]).max() < TOL
    assert np.abs(plain.alpha - g[f"f{frame}_alpha_img"]).max() < TOL
    hit = g[f"f{frame}_alpha_img"] >= 1e-3
    assert np.abs(plain.depth[hit] - g[f"f{frame}_depth"][hit]).max() < TOL
    assert np.all(plain.depth[~hit] == 1e9)


def test_cache_frame_mismatch(cuda):
    g = load("cache_d3")
    tree = tree_from(g)
    cache = vv.build_frame_cache(tree, 0)
    with pytest.raises(ValueError, match="cache built for frame 0"):
        vv.render_rays(tree, g["origins"], g["dirs"], 2, cache=cache)


def test_frame_out_of_range(cuda):
    g = load("cache_d3")
    tree = tree_from(g)
    with pytest.raises(ValueError, match="frame 99"):
        vv.render(tree, camera_from(g), 99)
    with pytest.raises(ValueError, match="out of range"):
        vv.build_frame_cache(tree, -1)


def test_config1(cuda):
    g = load("cfg1")
    tree = synthetic.shell_tree(depth=7, n_max=1, frames=16, seed=0)
    _check_rays(tree, g["origins"], g["dirs"], int(g["frame"]), g)
    cam = synthetic.bench_camera(64, 64)
    layer = vv.render(tree, cam, int(g["frame"]))
    assert np.abs(layer.rgb - g["rgb"]).max() < TOL
    assert np.abs(layer.alpha - g["alpha_img"]).max() < TOL
    hit = g["alpha_img"] >= 1e-3
    assert np.abs(layer.depth[hit] - g["depth"][hit]).max() < TOL
    start, leaf, t0, t1 = vv.collect_segments(tree, g["origins"], g["dirs"])
    _exact(leaf, g["seg_leaf"])
    _exact(t0, g["seg_t0"])


@pytest.mark.parametrize("frame", [0, 2])
@pytest.mark.parametrize("ew", [1.0, 0.4])
def test_edits(cuda, frame, ew):
    g = load("edits_d3")
    tree = tree_from(g)
    p, a, t = vv.render_rays(tree, g["origins"], g["dirs"], frame, vv.RenderOptions(edit_weight=ew))
    pre = f"f{frame}_w{int(ew * 10)}_"
    assert np.abs(a - g[pre + "alpha"]).max() <= 1e-12
    assert np.abs(t - g[pre + "tbar"]).max() <= 1e-9
    assert np.abs(p - g[pre + "premult"]).max() <= TOL


@pytest.mark.parametrize("n_max", [0, 3])
def test_other_truncations(cuda, n_max):
    g = load(f"nmax{n_max}")
    _check_rays(tree_from(g), g["origins"], g["dirs"], int(g["frame"]), g)


def test_scene_against_reference(cuda):
    g = load("scene")
    ta, tb = tree_from(g, "ta_"), tree_from(g, "tb_")
    cam = camera_from(g)

    def tr(x, y, z):
        m = np.eye(4)
        m[:3, 3] = [x, y, z]
        return m

    scale = np.diag([1.3, 1.3, 1.3, 1.0]) @ tr(-0.3, 0.1, 0.0)
    insts = [
        vv.SceneInstance(name="a", tree=ta, affine=tr(0.0, 0.0, 0.0)),
        vv.SceneInstance(name="b", tree=tb, affine=tr(1.2, 0.3, 0.0), timemap=vv.TimeMap.parse("shift(2)")),
        vv.SceneInstance(name="c", tree=ta, affine=scale, timemap=vv.TimeMap.parse("reverse")),
        vv.SceneInstance(name="d", tree=tb, affine=tr(-1.1, 0.4, 0.2), yaw_rate=15.0),
    ]
    scene = vv.Scene(instances=insts, background=np.array([0.1, 0.12, 0.2]))
    for gf in (0, 3):
        img = vv.render_scene(scene, cam, gf)
        assert np.abs(img - g[f"g{gf}_image"]).max() < TOL
        img2, blended, layers = vv.render_scene(scene, cam, gf, want_layers=True)
        assert np.abs(img2 - g[f"g{gf}_image"]).max() < TOL
        for i, l in enumerate(layers):
            assert np.abs(np.asarray(l.alpha) - g[f"g{gf}_layer{i}_alpha"]).max() < TOL
    single = vv.Scene(instances=[insts[2]], background=np.array([0.1, 0.12, 0.2]))
    assert np.abs(vv.render_scene(single, cam, 1) - g["single_image"]).max() < TOL


@pytest.mark.parametrize("depth,fill,seed", [(5, 0.3, 1), (6, 0.05, 2), (4, 0.9, 3), (3, 0.5, 4), (2, 0.6, 5),
                                             (1, 0.7, 6), (7, 0.02, 7)])
def test_random_trees_vs_oracle(cuda, depth, fill, seed):
    rng = np.random.default_rng(seed)
    res = 1 << depth
    coords = np.argwhere(rng.random((res, res, res)) < fill)
    k = 14
    data = rng.normal(scale=0.5, size=(len(coords), 2 * 7 + 3 * k)).astype(np.float32)
    data[:, 0] = rng.uniform(0.5, 60.0, len(coords))
    tree = vv.VOctree.from_cells(coords, data, vv.make_bump_bases(5, 7), 2, depth=depth)
    n = 4000
    o = rng.uniform(-1.0, 2.0, (n, 3))
    tgt = rng.uniform(0.1, 0.9, (n, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    ref = oracle.render_rays(tree, o, d, 3, visits=True)
    used, start, leaf = vv.render_ray_visits(tree, o, d, 3)
    _exact(used, ref["used"])
    _exact(leaf, ref["visit_leaf"])
    p, a, t, st = vv.render_rays(tree, o, d, 3, stats=True)
    _exact(st["node_pops"], ref["pops"], "node pops")
    _exact(st["shaded"], ref["shaded"], "shaded")
    assert np.abs(a - ref["alpha"]).max() <= 1e-12
    assert np.abs(p - ref["premult"]).max() <= TOL


def test_deep_tree_wide_stack(cuda):
    """depth 11 (> 9) exercises the 16-byte stack entries."""
    rng = np.random.default_rng(9)
    depth = 11
    res = 1 << depth
    centers = rng.integers(0, res - 64, (6, 3))
    coords = np.unique(np.concatenate([c + rng.integers(0, 64, (3000, 3)) for c in centers]), axis=0)
    data = rng.normal(scale=0.5, size=(len(coords), 2 * 3 + 3 * 5)).astype(np.float32)
    data[:, 0] = rng.uniform(100.0, 3000.0, len(coords))
    tree = vv.VOctree.from_cells(coords, data, vv.make_bump_bases(4, 3), 1, depth=depth)
    n = 3000
    o = rng.uniform(-0.5, 1.5, (n, 3))
    tgt = (centers[rng.integers(0, 6, n)] + 32) / res
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    ref = oracle.render_rays(tree, o, d, 1, visits=True)
    used, start, leaf = vv.render_ray_visits(tree, o, d, 1)
    assert ref["used"].sum() > 1000
    _exact(used, ref["used"])
    _exact(leaf, ref["visit_leaf"])
    start_g, leaf_g, t0_g, t1_g = vv.collect_segments(tree, o, d)
    start_r, leaf_r, t0_r, t1_r = oracle.collect_segments(tree, o, d)
    _exact(leaf_g, leaf_r)
    _exact(t0_g, t0_r)
    _exact(t1_g, t1_r)


def test_empty_tree(cuda):
    tree = vv.VOctree.from_cells(np.zeros((0, 3), int), np.zeros((0, 2 * 3 + 15), np.float32),
                                 vv.make_bump_bases(4, 3), 1, depth=2)
    cam = vv.Camera.look_at([2.0, 0.5, 0.5], [0.5, 0.5, 0.5], width=16, height=16)
    layer = vv.render(tree, cam, 0)
    assert np.all(layer.alpha == 0.0) and np.all(layer.rgb == 0.0) and np.all(layer.depth == 1e9)


def test_determinism(cuda):
    g = load("cache_d3")
    tree = tree_from(g)
    cam = camera_from(g)
    a = vv.render(tree, cam, 1)
    b = vv.render(tree, cam, 1)
    _exact(a.rgb, b.rgb)
    _exact(a.depth, b.depth)


def test_camera_rays_vs_host(cuda):
    """GPU-generated camera rays vs host Camera.rays: image within tolerance, and
    the fraction of rays whose visit lists agree with the host-ray oracle."""
    tree = synthetic.shell_tree(depth=7, n_max=1, frames=16, seed=0)
    cam = synthetic.bench_camera(160, 90)
    o, d = cam.rays()
    ref = oracle.render_rays(tree, o, d, 5)
    rgb, alpha, depth = oracle.finalize(ref["premult"], ref["alpha"], ref["tbar"])
    layer = vv.render(tree, cam, 5)
    assert np.abs(layer.rgb.reshape(-1, 3) - rgb).max() < TOL
    assert np.abs(layer.alpha.reshape(-1) - alpha).max() < TOL
    hit = alpha >= 1e-3
    assert np.abs(layer.depth.reshape(-1)[hit] - depth[hit]).max() < TOL


@pytest.mark.parametrize("depth", [2, 3, 6])
def test_dense_tree_full_stack(cuda, depth):
    """Every cell occupied and no early stop: oblique rays cross four children
    at every internal node, so the traversal stack reaches its bound
    (3 entries per level above the current node, stack_cap in vv_device.cuh).
    Visit lists and segments bit-exact, camera image within tolerance."""
    rng = np.random.default_rng(40 + depth)
    res = 1 << depth
    coords = np.argwhere(np.ones((res, res, res), bool))
    k = vv.hh.basis_count(1)
    data = rng.normal(scale=0.5, size=(len(coords), 2 * 3 + 3 * k)).astype(np.float32)
    data[:, 0] = rng.uniform(0.01, 0.05, len(coords)).astype(np.float32)
    tree = vv.VOctree.from_cells(coords, data, vv.make_bump_bases(4, 3), 1, depth=depth)
    n = 4000
    o = rng.uniform(-1.0, 2.0, (n, 3))
    o[:, rng.integers(0, 3)] = -0.75  # start outside the box
    d = rng.uniform(0.2, 0.8, 3) + rng.uniform(-0.1, 0.1, (n, 3))
    d *= np.where(o > 0.5, -1.0, 1.0)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    ref = oracle.render_rays(tree, o, d, 1, early_stop=0.0, visits=True)
    used, start, leaf = vv.render_ray_visits(tree, o, d, 1, vv.RenderOptions(early_stop=0.0))
    assert ref["used"].max() >= 3 * (depth - 1)
    _exact(used, ref["used"], "visit counts")
    _exact(leaf, ref["visit_leaf"], "visited leaves")
    start_g, leaf_g, t0_g, t1_g = vv.collect_segments(tree, o, d)
    start_r, leaf_r, t0_r, t1_r = oracle.collect_segments(tree, o, d)
    _exact(leaf_g, leaf_r)
    _exact(t0_g, t0_r)
    cam = vv.Camera.look_at([1.9, 1.6, -0.7], [0.5, 0.5, 0.5], width=96, height=64)
    co, cd = cam.rays()
    ref = oracle.render_rays(tree, co, cd, 2)
    rgb, alpha, _ = oracle.finalize(ref["premult"], ref["alpha"], ref["tbar"])
    layer = vv.render(tree, cam, 2)
    assert np.abs(layer.rgb.reshape(-1, 3) - rgb).max() < TOL
    assert np.abs(layer.alpha.reshape(-1) - alpha).max() < TOL


@pytest.mark.parametrize("name", ["cache_d3", "edits_d3"])
def test_decode_modes_bitwise_equal(cuda, name):
    """per_sample / per_frame / lazy leaf decoding give bitwise-identical
    renders (the reference's cached == uncached guarantee, render.py:14-17)."""
    g = load(name)
    tree = tree_from(g)
    o, d = g["origins"], g["dirs"]
    outs = {}
    for mode in ("per_sample", "per_frame", "auto"):
        outs[mode] = vv.render_rays(tree, o, d, 2, vv.RenderOptions(frame_slice=mode), stats=True)
    for mode in ("per_frame", "auto"):
        for a, b in zip(outs["per_sample"][:3], outs[mode][:3]):
            _exact(a, b, mode)
        _exact(outs["per_sample"][3]["sample_count"], outs[mode][3]["sample_count"], mode)


def test_decode_modes_config1_images(cuda):
    tree = synthetic.shell_tree(depth=7, n_max=1, frames=16, seed=0)
    cam = synthetic.bench_camera(96, 64)
    imgs = [vv.render(tree, cam, 5, vv.RenderOptions(frame_slice=m)) for m in ("per_sample", "per_frame", "auto")]
    for other in imgs[1:]:
        _exact(imgs[0].rgb, other.rgb)
        _exact(imgs[0].alpha, other.alpha)
        _exact(imgs[0].depth, other.depth)


def test_render_sequence_matches_render(cuda):
    tree = synthetic.shell_tree(depth=7, n_max=1, frames=16, seed=0)
    cam = synthetic.bench_camera(80, 48)
    frames = [3, 4, 5, 9, 0]
    seq = [l for l in vv.render_sequence(tree, cam, frames)]
    assert len(seq) == len(frames)
    for f, l in zip(frames, seq):
        ref = vv.render(tree, cam, f)
        _exact(l.rgb, ref.rgb)
        _exact(l.alpha, ref.alpha)
        _exact(l.depth, ref.depth)


def test_render_sequence_reuse_interleave_abandon(cuda):
    """Cached playback state: repeated calls, an abandoned generator and two
    interleaved generators on one device all still yield render()'s images."""
    tree = synthetic.shell_tree(depth=7, n_max=1, frames=16, seed=1)
    cam = synthetic.bench_camera(64, 40)
    ref = {f: vv.render(tree, cam, f) for f in range(8)}

    def same(l, f):
        _exact(l.rgb, ref[f].rgb)
        _exact(l.alpha, ref[f].alpha)
        _exact(l.depth, ref[f].depth)

    g = vv.render_sequence(tree, cam, [0, 1, 2, 3])
    same(next(g), 0)
    del g  # abandoned with a copy possibly in flight
    for _ in range(2):
        for f, l in zip([4, 5, 6], vv.render_sequence(tree, cam, [4, 5, 6])):
            same(l, f)
    a = vv.render_sequence(tree, cam, [0, 2, 4, 6])
    b = vv.render_sequence(tree, cam, [1, 3, 5, 7])
    for (fa, la), (fb, lb) in zip(zip([0, 2, 4, 6], a), zip([1, 3, 5, 7], b)):
        same(la, fa)
        same(lb, fb)


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["voct", "voct_edits"])
def test_load_device_matches_host_path(cuda, key):
    """.voct straight to the device (vv_voct_upload) renders bitwise like
    VOctree.from_bytes + upload, edits included."""
    g = load("voct")
    data = bytes(g[key])
    host = vv.VOctree.from_bytes(data)
    dev = vv.DeviceTree.from_voct(data)
    assert (dev.n_leaves, dev.depth, dev.frames, dev.has_edits) == (host.n_leaves, host.depth, host.frames,
                                                                    host.has_edits)
    cam = vv.Camera.look_at([2.1, -0.7, 1.5], [0.5, 0.5, 0.5], width=24, height=20)
    for f in (0, 2):
        a = vv.render(host, cam, f)
        b = vv.render(dev, cam, f)
        _exact(a.rgb, b.rgb)
        _exact(a.alpha, b.alpha)
        _exact(a.depth, b.depth)
    with pytest.raises(vv.ChecksumError):
        bad = bytearray(data)
        bad[300] ^= 4
        vv.DeviceTree.from_voct(bytes(bad))


@pytest.mark.gpu
@pytest.mark.parametrize("depth", [9, 11])
def test_deep_scene_launch(cuda, depth):
    """Deep trees in the fused scene kernel: traversal shared memory + the
    8 KB of staged basis rows exceed 48 KB per block (opt-in path)."""
    rng = np.random.default_rng(depth)
    res = 1 << depth
    coords = np.unique(rng.integers(res // 4, 3 * res // 4, (3000, 3)), axis=0)
    k = 14
    data = rng.normal(scale=0.5, size=(len(coords), 2 * 7 + 3 * k)).astype(np.float32)
    data[:, 0] = rng.uniform(50.0, 400.0, len(coords))
    tree = vv.VOctree.from_cells(coords, data, vv.make_bump_bases(4, 7), 2, depth=depth)
    m = np.eye(4)
    m[:3, 3] = [0.4, 0.1, 0.0]
    scene = vv.Scene(instances=[vv.SceneInstance(name="a", tree=tree),
                                vv.SceneInstance(name="b", tree=tree, affine=m)])
    cam = vv.Camera.look_at([0.6, -2.5, 1.2], [0.6, 0.5, 0.5], width=40, height=32)
    fused = vv.render_scene(scene, cam, 1)
    host, _, _ = vv.render_scene(scene, cam, 1, want_layers=True)
    assert np.abs(fused - host).max() < 1e-4


def _outs(torch, h, w, k):
    return [(torch.empty((h, w, 3), device="cuda"), torch.empty((h, w), device="cuda"),
             torch.empty((h, w), device="cuda")) for _ in range(k)]


@pytest.mark.gpu
@pytest.mark.parametrize("n_max,k", [(0, 2), (1, 3), (2, 4), (3, 2), (2, 3)])
def test_frames_share_one_walk_bitwise(cuda, n_max, k):
    """render_frames_into (several frames, one walk) == render_into per frame, bitwise."""
    import torch

    rng = np.random.default_rng(40 + n_max)
    res = 1 << 6
    coords = np.argwhere(rng.random((res, res, res)) < 0.08)
    kk = (n_max + 1) * (n_max + 2) * (2 * n_max + 3) // 6
    data = rng.normal(scale=0.5, size=(len(coords), 2 * 5 + 3 * kk)).astype(np.float32)
    data[:, 0] = rng.uniform(5.0, 60.0, len(coords))
    tree = vv.VOctree.from_cells(coords, data, vv.make_bump_bases(6, 5), n_max, depth=6)
    cam = vv.Camera.look_at([1.8, -0.9, 1.3], [0.5, 0.5, 0.5], width=96, height=72)
    frames = [5, 0, 3, 3][:k]  # any order, repeats allowed
    outs, refs = _outs(torch, 72, 96, k), _outs(torch, 72, 96, k)
    vv.render_frames_into(tree, cam, frames, outs)
    for f, r in zip(frames, refs):
        vv.render_into(tree, cam, f, *r)
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        for a, b in zip(o, r):
            assert torch.equal(a, b)


@pytest.mark.gpu
def test_frames_share_one_walk_with_edits(cuda):
    import torch

    g = load("edits_d3")
    tree = tree_from(g)
    cam = vv.Camera.look_at([2.1, -0.7, 1.5], [0.5, 0.5, 0.5], width=40, height=40)
    frames = [0, 2, 5]  # inside and outside the edit windows
    for ew in (1.0, 0.4):
        opts = vv.RenderOptions(edit_weight=ew, frame_slice="per_frame")
        outs, refs = _outs(torch, 40, 40, 3), _outs(torch, 40, 40, 3)
        vv.render_frames_into(tree, cam, frames, outs, opts)
        for f, r in zip(frames, refs):
            vv.render_into(tree, cam, f, *r, opts)
        torch.cuda.synchronize()
        assert all(torch.equal(a, b) for o, r in zip(outs, refs) for a, b in zip(o, r))


@pytest.mark.gpu
def test_frames_per_sample_fallback(cuda):
    """A tree small on screen decodes per sample: frames render one by one, same images."""
    import torch

    tree = synthetic.shell_tree(depth=7, n_max=1, frames=16, seed=0)
    cam = vv.Camera.look_at([6.0, 5.0, 4.0], [0.5, 0.5, 0.5], width=128, height=96)
    outs, refs = _outs(torch, 96, 128, 2), _outs(torch, 96, 128, 2)
    vv.render_frames_into(tree, cam, [1, 7], outs)
    for f, r in zip([1, 7], refs):
        vv.render_into(tree, cam, f, *r)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for o, r in zip(outs, refs) for a, b in zip(o, r))


@pytest.mark.gpu
def test_full_size_config2(cuda):
    """BASELINE configs[1] at full size (depth 9, 3,557,912 leaves, 1080p):
    visits / sample counts bit-exact against the oracle on a random pixel
    sample; the fused camera kernel agrees with render_rays on those pixels;
    shared-walk playback is bitwise equal to per-frame renders."""
    import torch

    tree = synthetic.shell_tree()
    cam = synthetic.bench_camera()
    o, d = cam.rays()
    rng = np.random.default_rng(99)
    idx = np.sort(rng.choice(len(o), 20000, replace=False))
    frame = 11
    ref = oracle.render_rays(tree, o[idx], d[idx], frame, visits=True)
    used, start, leaf = vv.render_ray_visits(tree, o[idx], d[idx], frame)
    _exact(used, ref["used"], "sample counts")
    _exact(leaf, ref["visit_leaf"], "visited leaves")
    assert (used > 0).sum() > 3000
    p, a, t = vv.render_rays(tree, o[idx], d[idx], frame)
    assert np.abs(a - ref["alpha"]).max() <= 1e-12
    assert np.abs(p - ref["premult"]).max() <= TOL
    layer = vv.render(tree, cam, frame)
    rgb, alpha, depth = oracle.finalize(p, a, t)
    assert np.abs(layer.rgb.reshape(-1, 3)[idx] - rgb).max() < TOL
    assert np.abs(layer.alpha.reshape(-1)[idx] - alpha).max() < TOL
    hit = alpha >= 1e-3
    assert np.abs(layer.depth.reshape(-1)[idx][hit] - depth[hit]).max() < TOL
    seq = list(vv.render_sequence(tree, cam, [frame, 12, 13, 29]))
    for f, l in zip([frame, 12, 13, 29], seq):
        r = vv.render(tree, cam, f)
        _exact(l.rgb, r.rgb)
        _exact(l.alpha, r.alpha)
        _exact(l.depth, r.depth)


@pytest.mark.gpu
@pytest.mark.parametrize("frames", [[2], [0, 5], [1, 1, 4], [3, 0, 2, 5]])
def test_slice_pass_several_frames_bitwise(cuda, frames):
    """build_frame_caches (one payload pass) == build_frame_cache per frame, bitwise."""
    g = load("cache_d3")
    tree = tree_from(g)
    frames = [f % tree.frames for f in frames]
    many = vv.build_frame_caches(tree, frames)
    for f, c in zip(frames, many):
        one = vv.build_frame_cache(tree, f)
        assert c.frame == f
        _exact(c.sigma.cpu().numpy(), one.sigma.cpu().numpy())
        _exact(c.q.cpu().numpy(), one.q.cpu().numpy())


@pytest.mark.gpu
def test_frames_share_one_walk_deep_and_empty(cuda):
    """Shared walk with wide (16-byte) stack entries (depth 11), and an empty tree."""
    import torch

    rng = np.random.default_rng(11)
    res = 1 << 11
    coords = np.unique(rng.integers(res // 3, 2 * res // 3, (4000, 3)), axis=0)
    data = rng.normal(scale=0.5, size=(len(coords), 2 * 5 + 3 * 5)).astype(np.float32)
    data[:, 0] = rng.uniform(100.0, 900.0, len(coords))
    tree = vv.VOctree.from_cells(coords, data, vv.make_bump_bases(4, 5), 1, depth=11)
    cam = vv.Camera.look_at([0.5, -1.5, 0.6], [0.5, 0.5, 0.5], width=64, height=48)
    opts = vv.RenderOptions(frame_slice="per_frame")
    outs, refs = _outs(torch, 48, 64, 3), _outs(torch, 48, 64, 3)
    vv.render_frames_into(tree, cam, [0, 1, 3], outs, opts)
    for f, r in zip([0, 1, 3], refs):
        vv.render_into(tree, cam, f, *r, opts)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for o, r in zip(outs, refs) for a, b in zip(o, r))
    assert float(outs[0][1].max()) > 0.0
    empty = vv.VOctree.from_cells(np.zeros((0, 3), np.int64), np.zeros((0, 25), np.float32),
                                  vv.make_bump_bases(4, 5), 1, depth=3)
    seq = list(vv.render_sequence(empty, cam, [0, 1, 2, 3]))
    assert len(seq) == 4 and all(np.all(l.alpha == 0.0) for l in seq)


def _sparse_bases(rng, frames=7, c=10):
    """Basis rows exercising the nonzero-chunk skipping (nz_chunks): only the
    constant column; a zero leading chunk; an all-zero row; a dense row; only
    the partial last chunk; negative entries; a single zero in each chunk."""
    a = np.zeros((frames, c), dtype=np.float32)
    a[0, 0] = 1.0
    a[1, [5, 9]] = [0.7, -0.4]
    a[3] = rng.normal(size=c)
    a[4, [8, 9]] = [0.9, 0.3]
    a[5, [0, 1, 6]] = [1.0, -0.8, 0.5]
    a[6] = rng.uniform(0.2, 1.0, c)
    a[6, [0, 5, 9]] = 0.0
    b = np.zeros_like(a)
    b[0] = rng.normal(size=c)
    b[1, 4] = 0.6
    b[3, [2, 3]] = [0.5, -0.5]
    b[4] = rng.normal(size=c)
    b[5, 9] = 1.2
    b[6] = rng.normal(size=c)
    return vv.TemporalBases(a, b)


@pytest.mark.parametrize("mode", ["per_sample", "per_frame"])
def test_sparse_basis_chunks_vs_oracle(cuda, mode):
    """The sigma / gamma sums skip float4 chunks whose basis entries are all
    zero: counts and visit lists stay exact, sigma bit-exact, colour within
    tolerance, against the oracle's full sums -- for every row shape."""
    rng = np.random.default_rng(11)
    depth, c, k = 5, 10, 14
    res = 1 << depth
    coords = np.argwhere(rng.random((res, res, res)) < 0.25)
    data = rng.normal(scale=0.6, size=(len(coords), 2 * c + 3 * k)).astype(np.float32)
    data[:, :c] *= 4.0  # sigma weights of both signs: some leaves dark in some frames
    bases = _sparse_bases(rng, 7, c)
    tree = vv.VOctree.from_cells(coords, data, bases, 2, depth=depth)
    n = 3000
    o = rng.uniform(-1.0, 2.0, (n, 3))
    d = rng.uniform(0.1, 0.9, (n, 3)) - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    opts = vv.RenderOptions(frame_slice=mode)
    for f in range(7):
        ref = oracle.render_rays(tree, o, d, f)
        p, a, t, st = vv.render_rays(tree, o, d, f, opts, stats=True)
        _exact(st["sample_count"], ref["used"], f"frame {f} counts")
        _exact(st["shaded"], ref["shaded"], f"frame {f} shaded")
        assert np.abs(a - ref["alpha"]).max() <= 1e-12, f
        assert np.abs(p - ref["premult"]).max() <= TOL, f
        sig, q = oracle.build_slice(tree, f)
        cache = vv.build_frame_cache(tree, f)
        _exact(cache.sigma.cpu().numpy(), sig, f"frame {f} slice sigma")
        assert np.abs(cache.q.cpu().numpy() - q).max() < 1e-5, f


def test_sparse_basis_multi_frame_slices_bitwise(cuda):
    """One multi-frame slice pass (union of the frames' chunk masks) gives
    every frame the records of its own single-frame pass."""
    rng = np.random.default_rng(12)
    depth, c, k = 5, 10, 14
    res = 1 << depth
    coords = np.argwhere(rng.random((res, res, res)) < 0.3)
    data = rng.normal(scale=0.6, size=(len(coords), 2 * c + 3 * k)).astype(np.float32)
    tree = vv.VOctree.from_cells(coords, data, _sparse_bases(rng, 7, c), 2, depth=depth)
    for group in ([0, 1], [2, 3, 4], [1, 4, 5, 6]):
        multi = vv.build_frame_caches(tree, group)
        for f, m in zip(group, multi):
            one = vv.build_frame_cache(tree, f)
            _exact(m.sigma.cpu().numpy(), one.sigma.cpu().numpy(), f"group {group} frame {f} sigma")
            _exact(m.q.cpu().numpy(), one.q.cpu().numpy(), f"group {group} frame {f} q")


def test_render_only_slices_dark_chunks_bitwise(cuda):
    """Render-internal slices (VV_SLICE_RENDER_ONLY) leave the colour of
    all-dark leaf chunks unwritten and skip their colour rows: on the cfg3
    motion generator (about 90% of leaves dark in any frame) render(),
    the shared-walk playback and the per-sample path stay bitwise equal to
    rendering from complete caches; exporting q from such a slice is refused."""
    import torch

    tree = synthetic.motion_tree(depth=7, frames=12)
    cam = synthetic.bench_camera(160, 96)
    h, w = cam.height, cam.width
    for f in (0, 5, 11):
        full = vv.build_frame_cache(tree, f)
        ref = vv.render(tree, cam, f, cache=full)
        for mode in ("per_frame", "per_sample"):
            img = vv.render(tree, cam, f, vv.RenderOptions(frame_slice=mode))
            _exact(img.rgb, ref.rgb, f"{mode} rgb {f}")
            _exact(img.alpha, ref.alpha, f"{mode} alpha {f}")
            _exact(img.depth, ref.depth, f"{mode} depth {f}")
        ro = vv.build_frame_caches(tree, [f], render_only=True)[0]
        _exact(ro.sigma.cpu().numpy(), full.sigma.cpu().numpy(), f"render-only sigma {f}")
        with pytest.raises(ValueError):
            ro.q
    frames = [2, 3, 4, 9]
    outs = [(torch.empty((h, w, 3), device=cuda), torch.empty((h, w), device=cuda), torch.empty((h, w), device=cuda))
            for _ in frames]
    vv.render_frames_into(tree, cam, frames, outs)
    torch.cuda.synchronize()
    for f, (r, a, d) in zip(frames, outs):
        ref = vv.render(tree, cam, f, cache=vv.build_frame_cache(tree, f))
        _exact(r.cpu().numpy(), ref.rgb, f"playback rgb {f}")
        _exact(a.cpu().numpy(), ref.alpha, f"playback alpha {f}")
        _exact(d.cpu().numpy(), ref.depth, f"playback depth {f}")


def test_slice_largest_stages_dense_c64_nmax3(cuda):
    """The widest slice stages: C = 64 dense A / B rows (16 chunks each) and
    n_max 3 (w_hh 30 x 3 floats) -- the launcher fits one warp per block.
    Sigma bit-exact and q within 1e-5 vs the oracle; 1..4-frame passes equal
    the single-frame pass bitwise; render-only slices render bitwise."""
    rng = np.random.default_rng(21)
    depth, c, k = 4, 64, 30
    res = 1 << depth
    coords = np.argwhere(rng.random((res, res, res)) < 0.5)
    data = rng.normal(scale=0.3, size=(len(coords), 2 * c + 3 * k)).astype(np.float32)
    a = rng.normal(scale=0.2, size=(6, c)).astype(np.float32)
    a[:, 0] = 1.0
    bases = vv.TemporalBases(a, rng.normal(scale=0.2, size=(6, c)).astype(np.float32))
    tree = vv.VOctree.from_cells(coords, data, bases, 3, depth=depth)
    for f in (0, 5):
        sig, q = oracle.build_slice(tree, f)
        one = vv.build_frame_cache(tree, f)
        _exact(one.sigma.cpu().numpy(), sig, f"sigma {f}")
        assert np.abs(one.q.cpu().numpy() - q).max() < 1e-5
    for group in ([1], [0, 3], [1, 2, 4], [0, 2, 3, 5]):
        multi = vv.build_frame_caches(tree, group)
        for f, m in zip(group, multi):
            one = vv.build_frame_cache(tree, f)
            _exact(m.sigma.cpu().numpy(), one.sigma.cpu().numpy(), f"group {group} sigma {f}")
            _exact(m.q.cpu().numpy(), one.q.cpu().numpy(), f"group {group} q {f}")
    cam = synthetic.bench_camera(72, 48)
    for f in (0, 4):
        ref = vv.render(tree, cam, f, cache=vv.build_frame_cache(tree, f))
        img = vv.render(tree, cam, f, vv.RenderOptions(frame_slice="per_frame"))
        _exact(img.rgb, ref.rgb, f"render-only rgb {f}")
        _exact(img.alpha, ref.alpha, f"render-only alpha {f}")


def test_no_device_memory_growth(cuda):
    """Repeated renders in every decode mode, slice caches and playback
    release their transient device memory (stream-ordered pool frees)."""
    import torch

    tree = synthetic.shell_tree(depth=7, n_max=1, frames=8, seed=5)
    cam = synthetic.bench_camera(96, 64)
    modes = ("auto", "per_sample", "per_frame")

    def work():
        for f in range(8):
            for m in modes:
                vv.render(tree, cam, f, vv.RenderOptions(frame_slice=m))
            c = vv.build_frame_cache(tree, f)
            vv.render(tree, cam, f, cache=c)
            del c
        for _ in vv.render_sequence(tree, cam, range(8)):
            pass
        torch.cuda.synchronize()

    work()  # pools and caches reach their steady size
    free0 = torch.cuda.mem_get_info(cuda)[0]
    for _ in range(5):
        work()
    free1 = torch.cuda.mem_get_info(cuda)[0]
    assert free0 - free1 < (64 << 20), f"device memory fell by {(free0 - free1) >> 20} MB"


def test_render_options_through_camera_kernel(cuda):
    """Non-default RenderOptions (alpha floor, far plane, early stop)
    through the fused camera kernel: within tolerance of the oracle's rays +
    the host finalize_layer, every decode mode bitwise alike."""
    tree = synthetic.shell_tree(depth=7, n_max=2, frames=6, seed=8)
    cam = synthetic.bench_camera(96, 64)
    opts = dict(alpha_floor=0.3, far_plane=7.5, early_stop=1e-3)
    o, d = cam.rays()
    for f in (1, 4):
        ref = oracle.render_rays(tree, o, d, f, early_stop=opts["early_stop"])
        host = vv.finalize_layer(ref["premult"], ref["alpha"], ref["tbar"], (cam.height, cam.width),
                                 vv.RenderOptions(**opts))
        imgs = [vv.render(tree, cam, f, vv.RenderOptions(frame_slice=m, **opts))
                for m in ("per_frame", "per_sample", "auto")]
        a0 = np.asarray(imgs[0].alpha)
        assert np.abs(np.asarray(imgs[0].rgb) - host.rgb).max() <= TOL
        assert np.abs(a0 - host.alpha).max() <= TOL
        hit = a0 >= opts["alpha_floor"]
        assert np.all(np.asarray(imgs[0].depth)[~hit] == np.float32(opts["far_plane"]))
        assert np.abs(np.asarray(imgs[0].depth)[hit] - np.asarray(host.depth)[hit]).max() <= TOL
        for other in imgs[1:]:
            _exact(other.rgb, imgs[0].rgb, f"frame {f} rgb across modes")
            _exact(other.alpha, imgs[0].alpha, f"frame {f} alpha across modes")
            _exact(other.depth, imgs[0].depth, f"frame {f} depth across modes")


@pytest.mark.parametrize("lo,side", [((-0.3, 0.2, 0.1), 1.7), ((0.5, -1.0, 0.25), 0.25), ((0.0, 0.0, 0.0), 4.0),
                                     ((0.1, 0.1, 0.1), 3.0e-3)])
def test_bbox_placement_vs_oracle(cuda, lo, side):
    """Trees placed off the unit cube: ray setup divides by a general side and
    multiplies by 1/side for a power-of-two side (exact either way) -- visit
    lists, counts and images against the oracle."""
    rng = np.random.default_rng(17)
    depth, c, k = 5, 6, 14
    res = 1 << depth
    coords = np.argwhere(rng.random((res, res, res)) < 0.2)
    data = rng.normal(scale=0.5, size=(len(coords), 2 * c + 3 * k)).astype(np.float32)
    data[:, 0] = rng.uniform(0.5, 30.0, len(coords)) / side
    tree = vv.VOctree.from_cells(coords, data, vv.make_bump_bases(4, c), 2, bbox_lo=lo, side=side, depth=depth)
    lo_ = np.asarray(lo)
    n = 3000
    o = lo_ + side * rng.uniform(-1.0, 2.0, (n, 3))
    d = lo_ + side * rng.uniform(0.2, 0.8, (n, 3)) - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    ref = oracle.render_rays(tree, o, d, 2, visits=True)
    used, start, leaf = vv.render_ray_visits(tree, o, d, 2)
    _exact(used, ref["used"], "counts")
    _exact(leaf, ref["visit_leaf"], "visits")
    p, a, t = vv.render_rays(tree, o, d, 2)
    assert np.abs(a - ref["alpha"]).max() <= 1e-12
    assert np.abs(p - ref["premult"]).max() <= TOL


def test_render_sequences_zipped_stereo(cuda):
    """Two playbacks live at once (the eyes of a stereo sequence, zipped):
    each gets a cached playback state of its own; every frame bitwise render()."""
    tree = synthetic.shell_tree(depth=7, n_max=1, frames=8, seed=3)
    eyes = [vv.Camera.look_at(e, [0.5, 0.5, 0.5], width=96, height=80) for e in ([1.7, 1.2, 0.9], [1.6, 1.35, 0.9])]
    frames = [0, 3, 5, 6, 1, 7, 2]
    for _ in range(2):  # second round: cached states reused
        got = list(zip(*[vv.render_sequence(tree, cam, frames) for cam in eyes]))
        assert len(got) == len(frames)
        for f, pair in zip(frames, got):
            for cam, layer in zip(eyes, pair):
                ref = vv.render(tree, cam, f)
                _exact(layer.rgb, ref.rgb, f"rgb {f}")
                _exact(layer.depth, ref.depth, f"depth {f}")
