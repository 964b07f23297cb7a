"""Multi-GPU tile paths on one GPU.

* packed tiles (vv_render_camera_tiles) of every shard, gathered shard-major
  and scattered by vv_unpack_tiles, reproduce render() bitwise;
* the fused direct form (vv_render_camera_tiles_direct) writes exactly its
  shard's pixels of the full image, bitwise equal to render(), and leaves
  every other pixel untouched;
* TileRenderer(mode="p2p") end to end with two processes on this GPU (gloo
  for the handle exchange and the barrier): rank 1 maps rank 0's planes
  through CUDA IPC and stores its tiles there; rank 0's frame equals
  render().  Two ranks sharing one GPU only check the plumbing: the peer
  stores go through the same device's memory, no kernel waits on another.
"""

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import synthetic
from paper_2202_06088_b200.distributed import TileRenderer, tile_mask_host

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
W, H, TILE = 208, 144, 64  # ragged: the last tile column/row is partial


def _tree():
    return synthetic.shell_tree(depth=7, n_max=1, frames=8, seed=3)


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def _eq(a, b, what):
    a, b = _np(a), _np(b)
    assert a.shape == b.shape, what
    assert np.array_equal(a, b, equal_nan=False), f"{what}: {np.count_nonzero(a != b)} mismatches"


@pytest.mark.parametrize("world", [1, 3])
def test_packed_tiles_gather_unpack_bitwise(cuda, world):
    import torch

    tree, cam = _tree(), synthetic.bench_camera(W, H)
    ref = vv.render(tree, cam, 5)
    slabs = []
    for s in range(world):
        tr = TileRenderer(W, H, TILE, rank=s, world=world, device=cuda)
        slabs.append(tr.render_slab(tree, cam, 5).clone())
    tr.all.copy_(torch.stack(slabs))
    rgb = torch.full((H, W, 3), float("nan"), device=cuda)
    alpha = torch.full((H, W), float("nan"), device=cuda)
    depth = torch.full((H, W), float("nan"), device=cuda)
    tr.unpack(rgb, alpha, depth)
    torch.cuda.synchronize()
    _eq(rgb, ref.rgb, "rgb")
    _eq(alpha, ref.alpha, "alpha")
    _eq(depth, ref.depth, "depth")


def test_direct_tiles_write_only_their_shard(cuda):
    import ctypes

    import torch

    from paper_2202_06088_b200 import _native
    from paper_2202_06088_b200.device import replica, stream_ptr

    tree, cam = _tree(), synthetic.bench_camera(W, H)
    ref = vv.render(tree, cam, 2)
    rep = replica(tree, cuda)
    rgb = torch.full((H, W, 3), float("nan"), device=cuda)
    alpha = torch.full((H, W), float("nan"), device=cuda)
    depth = torch.full((H, W), float("nan"), device=cuda)
    oc, cd = vv.RenderOptions().c_struct(), cam.desc()
    world = 3
    covered = np.zeros((H, W), dtype=bool)
    for s in range(world):
        _native.check(_native.lib().vv_render_camera_tiles_direct(
            rep.handle, 2, None, ctypes.byref(oc), ctypes.byref(cd), TILE, s, world, rgb.data_ptr(),
            alpha.data_ptr(), depth.data_ptr(), 0, stream_ptr(cuda)))
        torch.cuda.synchronize()
        covered |= tile_mask_host(s, world, W, H, TILE)
        a = _np(alpha)
        assert np.array_equal(np.isnan(a), ~covered), f"shard {s} wrote outside its tiles"
        _eq(a[covered], _np(ref.alpha)[covered], f"alpha after shard {s}")
    assert covered.all()
    _eq(rgb, ref.rgb, "rgb")
    _eq(depth, ref.depth, "depth")
    with pytest.raises(ValueError):  # tile not a multiple of 16
        _native.check(_native.lib().vv_render_camera_tiles_direct(
            rep.handle, 2, None, ctypes.byref(oc), ctypes.byref(cd), 24, 0, 1, rgb.data_ptr(), None, None, 0,
            stream_ptr(cuda)))


def test_p2p_renderer_world1(cuda):
    tree, cam = _tree(), synthetic.bench_camera(W, H)
    tr = TileRenderer(W, H, TILE, rank=0, world=1, device=cuda, mode="p2p")
    try:
        for f in (1, 4, 6):  # alternating slots
            out = tr.render_frame(tree, cam, f)
            ref = vv.render(tree, cam, f)
            _eq(out.rgb, ref.rgb, f"rgb frame {f}")
            _eq(out.alpha, ref.alpha, f"alpha frame {f}")
            _eq(out.depth, ref.depth, f"depth frame {f}")
        with pytest.raises(ValueError):
            tr.render_frame(tree, synthetic.bench_camera(W + 16, H), 0)
    finally:
        tr.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", ["p2p", "regions"])
def test_p2p_renderer_two_processes_ipc(cuda, mode):
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   PYTHONPATH=str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", ""))
        procs.append(subprocess.Popen([sys.executable, str(ROOT / "tests" / "p2p_worker.py"), mode], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=300)[0])
        except subprocess.TimeoutExpired:
            p.kill()
            outs.append(p.communicate()[0])
    for r, (p, o) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, f"rank {r} failed:\n{o[-3000:]}"
    assert "P2P_OK" in outs[0], outs[0][-2000:]


def test_back_to_back_renders_same_outputs_ordered(cuda):
    """Programmatic dependent launch lets a render start during the previous
    kernel's tail; every output write waits for it.  Many frames rendered
    into the SAME buffers back to back (no sync, mixed decode modes, tile
    shards in direct mode) must leave exactly the last frame's images."""
    import ctypes

    import torch

    from paper_2202_06088_b200 import _native
    from paper_2202_06088_b200.device import replica, stream_ptr

    tree, cam = _tree(), synthetic.bench_camera(W, H)
    rgb = torch.zeros((H, W, 3), device=cuda)
    alpha = torch.zeros((H, W), device=cuda)
    depth = torch.zeros((H, W), device=cuda)
    modes = ("per_frame", "per_sample", "auto")
    for i in range(24):
        vv.render_into(tree, cam, i % tree.frames, rgb, alpha, depth, vv.RenderOptions(frame_slice=modes[i % 3]))
    last = 23 % tree.frames
    torch.cuda.synchronize()
    ref = vv.render(tree, cam, last)
    _eq(rgb, ref.rgb, "rgb after back-to-back renders")
    _eq(alpha, ref.alpha, "alpha after back-to-back renders")
    _eq(depth, ref.depth, "depth after back-to-back renders")
    # tile shards of alternating frames into one image: the last pass per shard wins
    rep = replica(tree, cuda)
    oc, cd = vv.RenderOptions().c_struct(), cam.desc()
    world = 3
    for rnd in range(4):
        f = (rnd * 5) % tree.frames
        for s in range(world):
            _native.check(_native.lib().vv_render_camera_tiles_direct(
                rep.handle, f, None, ctypes.byref(oc), ctypes.byref(cd), TILE, s, world, rgb.data_ptr(),
                alpha.data_ptr(), depth.data_ptr(), 0, stream_ptr(cuda)))
    torch.cuda.synchronize()
    ref = vv.render(tree, cam, (3 * 5) % tree.frames)
    _eq(rgb, ref.rgb, "rgb after tile rounds")
    _eq(alpha, ref.alpha, "alpha after tile rounds")


@pytest.mark.parametrize("tile,world", [(16, 2), (32, 5), (128, 2)])
def test_direct_tiles_sizes_and_worlds(cuda, tile, world):
    """Direct tile rendering for other tile sizes and shard counts (ragged
    image): the shards' union is render() bitwise."""
    import ctypes

    import torch

    from paper_2202_06088_b200 import _native
    from paper_2202_06088_b200.device import replica, stream_ptr

    w, h = 200, 136
    tree, cam = _tree(), synthetic.bench_camera(w, h)
    ref = vv.render(tree, cam, 3)
    rep = replica(tree, cuda)
    rgb = torch.full((h, w, 3), float("nan"), device=cuda)
    alpha = torch.full((h, w), float("nan"), device=cuda)
    depth = torch.full((h, w), float("nan"), device=cuda)
    oc, cd = vv.RenderOptions().c_struct(), cam.desc()
    for s in range(world):
        _native.check(_native.lib().vv_render_camera_tiles_direct(
            rep.handle, 3, None, ctypes.byref(oc), ctypes.byref(cd), tile, s, world, rgb.data_ptr(),
            alpha.data_ptr(), depth.data_ptr(), 0, stream_ptr(cuda)))
    torch.cuda.synchronize()
    _eq(rgb, ref.rgb, "rgb")
    _eq(alpha, ref.alpha, "alpha")
    _eq(depth, ref.depth, "depth")


# ------------------------------------------------------------------ regions
def _region_union(tree, cam, frame, bands, opts=None):
    """Render each band into NaN planes; check each band writes only its rows."""
    import torch

    from paper_2202_06088_b200.distributed import render_region

    h, w = cam.height, cam.width
    rgb = torch.full((h, w, 3), float("nan"), device="cuda")
    alpha = torch.full((h, w), float("nan"), device="cuda")
    depth = torch.full((h, w), float("nan"), device="cuda")
    from paper_2202_06088_b200.distributed import block_order, pixel_costs

    costs = pixel_costs(tree, cam, frame)
    for k in range(len(bands) - 1):
        rect = (0, bands[k], w, bands[k + 1])
        order = block_order(costs, rect) if k % 2 else None  # both launch orders
        render_region(tree, cam, frame, rect, rgb, alpha, depth, opts, order=order)
        torch.cuda.synchronize()
        a = _np(alpha)
        assert not np.isnan(a[:bands[k + 1]]).any() and np.isnan(a[bands[k + 1]:]).all(), f"band {k}"
    return rgb, alpha, depth


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_region_bands_bitwise(cuda, world):
    """Row bands balanced on measured row costs: each band slices only the
    leaf chunks its pixels can reach (chunk culling) and writes only its rows;
    their union is render() bitwise (ragged image, every decode mode)."""
    from paper_2202_06088_b200.distributed import band_plan, row_costs

    tree, cam = _tree(), synthetic.bench_camera(W, H)
    bands = band_plan(row_costs(tree, cam, 2), world)
    assert bands[0] == 0 and bands[-1] == H and all(a <= b for a, b in zip(bands, bands[1:]))
    for mode in ("per_frame", "auto", "per_sample"):
        opts = vv.RenderOptions(frame_slice=mode)
        ref = vv.render(tree, cam, 2, opts)
        rgb, alpha, depth = _region_union(tree, cam, 2, bands, opts)
        _eq(rgb, ref.rgb, f"{mode} rgb")
        _eq(alpha, ref.alpha, f"{mode} alpha")
        _eq(depth, ref.depth, f"{mode} depth")


def test_region_rectangles_and_inside_camera(cuda):
    """Arbitrary rectangles (2D split), and an eye inside the tree's cube
    (chunk corners behind the camera are kept conservatively)."""
    import torch

    from paper_2202_06088_b200.distributed import render_region

    tree = _tree()
    opts = vv.RenderOptions(frame_slice="per_frame")
    for cam in (synthetic.bench_camera(W, H),
                vv.Camera.look_at([0.5, 0.45, 0.5], [1.0, 0.9, 0.7], width=W, height=H, focal=0.6 * W)):
        ref = vv.render(tree, cam, 5, opts)
        rgb = torch.full((H, W, 3), float("nan"), device=cuda)
        alpha = torch.full((H, W), float("nan"), device=cuda)
        depth = torch.full((H, W), float("nan"), device=cuda)
        xs, ys = (0, 48, 130, W), (0, 40, 96, H)
        for i in range(3):
            for j in range(3):
                render_region(tree, cam, 5, (xs[i], ys[j], xs[i + 1], ys[j + 1]), rgb, alpha, depth, opts)
        torch.cuda.synchronize()
        _eq(rgb, ref.rgb, "rect rgb")
        _eq(alpha, ref.alpha, "rect alpha")
        _eq(depth, ref.depth, "rect depth")


@pytest.mark.parametrize("gen", ["shell", "motion"])
def test_region_bands_full_size(cuda, gen):
    """cfg2 / cfg3 at 1080p in 8 measured bands: bitwise equal to render()
    (cfg3 adds the node masks, with unlisted leaves treated as dark)."""
    from paper_2202_06088_b200.distributed import band_plan, row_costs

    tree = synthetic.shell_tree() if gen == "shell" else synthetic.motion_tree()
    cam = synthetic.bench_camera()
    bands = band_plan(row_costs(tree, cam, 4), 8)
    for f in (4, 17):
        ref = vv.render(tree, cam, f)
        rgb, alpha, depth = _region_union(tree, cam, f, bands)
        _eq(rgb, ref.rgb, f"{gen} rgb {f}")
        _eq(alpha, ref.alpha, f"{gen} alpha {f}")
        _eq(depth, ref.depth, f"{gen} depth {f}")


# ------------------------------------------------------------------ camera plans
def test_camera_plan_bitwise_over_frames_and_sizes(cuda):
    """Renders through a CameraPlan (persistent warps in the previous frame's
    cost order) are bitwise render(): first frame (no order yet), later
    frames (learned order), a resized camera (plan re-sized), a region, and
    a second tree sharing the plan (any valid order schedules correctly)."""
    import torch

    tree, other = _tree(), synthetic.shell_tree(depth=6, n_max=2, frames=5, seed=9)
    plan = vv.CameraPlan(cuda)
    for w, h in ((W, H), (W, H), (128, 96), (W, H)):
        cam = synthetic.bench_camera(w, h)
        for f in (0, 3, 7):
            for t in (tree, other):
                f_ = f % t.frames
                outs = [torch.full((h, w, 3), float("nan"), device=cuda), torch.full((h, w), float("nan"), device=cuda),
                        torch.full((h, w), float("nan"), device=cuda)]
                vv.render_into(t, cam, f_, *outs, plan=plan)
                ref = vv.render(t, cam, f_)
                torch.cuda.synchronize()
                _eq(outs[0], ref.rgb, f"plan rgb {w}x{h} f{f_}")
                _eq(outs[1], ref.alpha, f"plan alpha {w}x{h} f{f_}")
                _eq(outs[2], ref.depth, f"plan depth {w}x{h} f{f_}")


def test_camera_plan_regions_renderer_world1(cuda):
    """TileRenderer(mode="regions") at world 1 (one band, planned) equals render()."""
    tree, cam = _tree(), synthetic.bench_camera(W, H)
    tr = TileRenderer(W, H, TILE, rank=0, world=1, device=cuda, mode="regions")
    try:
        for f in (1, 4, 6, 2):
            out = tr.render_frame(tree, cam, f)
            ref = vv.render(tree, cam, f)
            _eq(out.rgb, ref.rgb, f"rgb frame {f}")
            _eq(out.depth, ref.depth, f"depth frame {f}")
    finally:
        tr.close()


def test_camera_plan_cfg3_masked(cuda):
    """Planned renders of the cfg3 motion tree (node masks on) at 1080p,
    bitwise equal to unplanned ones across a frame sweep."""
    import torch

    tree, cam = synthetic.motion_tree(), synthetic.bench_camera()
    plan = vv.CameraPlan(cuda)
    h, w = cam.height, cam.width
    for f in (0, 7, 30, 31, 59):
        outs = [torch.empty((h, w, 3), device=cuda), torch.empty((h, w), device=cuda), torch.empty((h, w), device=cuda)]
        vv.render_into(tree, cam, f, *outs, plan=plan)
        ref = vv.render(tree, cam, f)
        torch.cuda.synchronize()
        _eq(outs[0], ref.rgb, f"cfg3 plan rgb {f}")
        _eq(outs[2], ref.depth, f"cfg3 plan depth {f}")


def test_render_to_host_banded_copies(cuda):
    """render() -> numpy copies 64-row bands behind the kernel (copy stream
    waiting on per-band counters): bitwise the device render, for ragged
    sizes, a frame taller than one band and back-to-back calls reusing
    pinned buffers."""
    import torch

    tree = _tree()
    for w, h in ((W, H), (97, 203), (1920, 1080)):
        cam = synthetic.bench_camera(w, h)
        for f in (2, 5):
            dev = vv.render(tree, cam, f, out="torch")
            host = vv.render(tree, cam, f)
            torch.cuda.synchronize()
            _eq(host.rgb, dev.rgb, f"rgb {w}x{h} f{f}")
            _eq(host.alpha, dev.alpha, f"alpha {w}x{h} f{f}")
            _eq(host.depth, dev.depth, f"depth {w}x{h} f{f}")


def test_camera_plan_coverage_reuse_and_invalidation(cuda):
    """A plan caches the chunk-box coverage of its (tree, camera): renders of
    the same view reuse it, a new camera or a new tree (even one allocated
    where a freed tree lived) rebuilds it -- bitwise render() every time."""
    import torch

    plan = vv.CameraPlan(cuda)
    cams = [synthetic.bench_camera(W, H),
            vv.Camera.look_at([-0.9, 1.6, 1.2], [0.5, 0.5, 0.5], width=W, height=H, focal=1.1 * W)]
    for it in range(3):
        tree = synthetic.shell_tree(depth=6, n_max=1, frames=6, seed=it)  # replaces the previous tree
        for cam in cams + cams[:1]:
            for f in (0, 4):
                out = [torch.empty((H, W, 3), device=cuda), torch.empty((H, W), device=cuda),
                       torch.empty((H, W), device=cuda)]
                vv.render_into(tree, cam, f, *out, plan=plan)
                ref = vv.render(tree, cam, f, out="torch")
                torch.cuda.synchronize()
                _eq(out[0], ref.rgb, f"rgb it{it} f{f}")
                _eq(out[1], ref.alpha, f"alpha it{it} f{f}")
                _eq(out[2], ref.depth, f"depth it{it} f{f}")
        del tree


def test_plans_with_eye_inside_and_grazing_views(cuda):
    """Coverage and occupied-box skipping are conservative: an eye inside the
    tree's cube (box corners behind it), a view from below with the tree half
    off-screen, and a narrow field of view on a cube edge -- planned renders
    (camera, playback) bitwise equal to unplanned ones."""
    import torch

    tree = _tree()
    cams = [vv.Camera.look_at([0.5, 0.45, 0.5], [1.0, 0.9, 0.7], width=W, height=H, focal=0.6 * W),
            vv.Camera.look_at([0.9, 0.2, -1.2], [0.9, 0.3, 0.5], width=W, height=H, focal=1.5 * W),
            vv.Camera.look_at([3.0, 3.1, 2.9], [1.0, 1.0, 0.5], width=W, height=H, focal=9.0 * W)]
    plan = vv.CameraPlan(cuda)
    for cam in cams:
        for f in (1, 6):
            out = [torch.empty((H, W, 3), device=cuda), torch.empty((H, W), device=cuda),
                   torch.empty((H, W), device=cuda)]
            vv.render_into(tree, cam, f, *out, plan=plan)
            ref = vv.render(tree, cam, f, vv.RenderOptions(frame_slice="per_sample"), out="torch")
            torch.cuda.synchronize()
            _eq(out[0], ref.rgb, "rgb")
            _eq(out[2], ref.depth, "depth")
        outs = [(torch.empty((H, W, 3), device=cuda), torch.empty((H, W), device=cuda),
                 torch.empty((H, W), device=cuda)) for _ in range(3)]
        vv.render_frames_into(tree, cam, [0, 3, 5], outs, vv.RenderOptions(frame_slice="per_frame"))
        torch.cuda.synchronize()
        for f, o in zip([0, 3, 5], outs):
            ref = vv.render(tree, cam, f, out="torch")
            _eq(o[0], ref.rgb, f"playback rgb {f}")
            _eq(o[1], ref.alpha, f"playback alpha {f}")
