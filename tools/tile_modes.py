"""Single-GPU emulation of one frame split across N GPUs.

Every rank's share of a 1080p frame is rendered here one after another on
this one GPU and timed alone (CUDA events, L2 flushed before each share);
the frame time at N GPUs is the slowest rank's share (the gather over
NVLink -- 20 B/px, stored by the render kernel itself in "regions" and
"p2p" modes -- is not included).  Two partitions:

* interleaved 64x64 tiles (tile_id % N == rank, vv_render_camera_tiles_direct):
  every rank decodes every leaf (whole-tree slice pass, or per sample);
* contiguous row bands balanced on measured row costs (TileRenderer
  mode="regions", vv_render_camera_region): each rank slices only the leaf
  chunks its band can reach.

    python tools/tile_modes.py [--tree shell|motion] [--worlds 1,2,4,8]
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import _native, synthetic  # noqa: E402
from paper_2202_06088_b200.device import replica, stream_ptr  # noqa: E402
from paper_2202_06088_b200.distributed import band_plan, pixel_costs, render_region  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tree", default="shell", choices=["shell", "motion"])
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--frames", type=int, default=8)
args = ap.parse_args()

dev = torch.device("cuda", 0)
tree = synthetic.motion_tree() if args.tree == "motion" else synthetic.shell_tree()
cam = synthetic.bench_camera()
h, w = cam.height, cam.width
rgb = torch.empty((h, w, 3), device=dev)
alpha = torch.empty((h, w), device=dev)
depth = torch.empty((h, w), device=dev)
flush = torch.empty(64 * 2**20, dtype=torch.float32, device=dev)
rep = replica(tree, dev)
T = tree.frames


def share_ms(fn):
    """Mean per-frame time of one rank's share (L2 flushed before each frame)."""
    for f in range(3):
        fn(f)
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(args.frames):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn((5 * i) % T)
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / args.frames


def tiles(world, rank):
    oc, cd = vv.RenderOptions().c_struct(), cam.desc()

    def fn(f):
        _native.check(_native.lib().vv_render_camera_tiles_direct(
            rep.handle, f, None, ctypes.byref(oc), ctypes.byref(cd), 64, rank, world, rgb.data_ptr(),
            alpha.data_ptr(), depth.data_ptr(), 0, stream_ptr(dev)))
    return fn


def bands(edges, rank, ordered=True):
    """ordered: the rank's own camera plan (what TileRenderer "regions" runs:
    persistent warps in its measured cost order, cached coverage); else the
    static row-major launch."""
    rect = (0, edges[rank], w, edges[rank + 1])
    plan = vv.CameraPlan(dev) if ordered else None
    return lambda f: render_region(tree, cam, f, rect, rgb, alpha, depth, plan=plan)


out = {"tree": args.tree, "single_gpu_frame_ms": round(share_ms(lambda f: vv.render_into(tree, cam, f, rgb, alpha,
                                                                                            depth)), 4)}
costs = pixel_costs(tree, cam, 0)
rows = costs.sum(dim=1).cpu().numpy()
for world in [int(x) for x in args.worlds.split(",")]:
    edges = band_plan(rows, world)
    band_ms = [share_ms(bands(edges, r)) for r in range(world)]
    plain_ms = [share_ms(bands(edges, r, False)) for r in range(world)]
    tile_ms = [share_ms(tiles(world, r)) for r in range(world)]
    out[f"n{world}"] = {
        "bands": {"edges": edges, "per_rank_ms": [round(x, 4) for x in band_ms], "frame_ms": round(max(band_ms), 4),
                  "efficiency": round(out["single_gpu_frame_ms"] / (world * max(band_ms)), 3),
                  "unordered_frame_ms": round(max(plain_ms), 4)},
        "tiles64": {"per_rank_ms": [round(x, 4) for x in tile_ms], "frame_ms": round(max(tile_ms), 4),
                    "efficiency": round(out["single_gpu_frame_ms"] / (world * max(tile_ms)), 3)},
    }
    print(json.dumps({f"n{world}": out[f"n{world}"]}), file=sys.stderr, flush=True)
print(json.dumps(out))
