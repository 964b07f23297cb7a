"""Render-kernel launch strategies for a full 1080p frame and for 8 row
bands of it (region renders), from one full-frame slice (cache), L2 flushed
before each kernel:

* static blocks in row-major order (the default image kernel);
* static blocks in cost order (LPT, costliest first: block_order);
* persistent warps pulling warp chunks from a counter (VV_CAM_QUEUE=1), in
  row-major or cost order.

    python tools/band_warm_probe.py [--tree shell|motion]
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402
from paper_2202_06088_b200.distributed import band_plan, block_order, pixel_costs, render_region  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tree", default="shell")
args = ap.parse_args()
tree = synthetic.motion_tree() if args.tree == "motion" else synthetic.shell_tree()
cam = synthetic.bench_camera()
h, w = cam.height, cam.width
rgb = torch.empty((h, w, 3), device="cuda")
alpha = torch.empty((h, w), device="cuda")
depth = torch.empty((h, w), device="cuda")
costs = pixel_costs(tree, cam, 0)
edges = band_plan(costs.sum(dim=1).cpu().numpy(), 8)
cache = vv.build_frame_cache(tree, 5)
flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")


def ev(fn, n=10):
    for _ in range(2):
        fn()
    tot = 0.0
    for _ in range(n):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return round(tot / n, 4)


rects = [(0, edges[r], w, edges[r + 1]) for r in range(8)]
orders = [block_order(costs, rc) for rc in rects]
full_rect = (0, 0, w, h)
full_order = block_order(costs, full_rect)
out = {"edges": edges}
for q in ("0", "1"):
    os.environ["VV_CAM_QUEUE"] = q
    tag = "queue" if q == "1" else "static"
    out[f"full_{tag}_rowmajor"] = ev(lambda: render_region(tree, cam, 5, full_rect, rgb, alpha, depth, cache=cache))
    out[f"full_{tag}_lpt"] = ev(lambda: render_region(tree, cam, 5, full_rect, rgb, alpha, depth, cache=cache,
                                                      order=full_order))
    for nm, od in (("rowmajor", [None] * 8), ("lpt", orders)):
        b = [ev(lambda r=r: render_region(tree, cam, 5, rects[r], rgb, alpha, depth, cache=cache, order=od[r]))
             for r in range(8)]
        out[f"bands_{tag}_{nm}"] = {"per_band": b, "max": max(b), "sum": round(sum(b), 4)}
del os.environ["VV_CAM_QUEUE"]
out["render_into_default"] = ev(lambda: vv.render_into(tree, cam, 5, rgb, alpha, depth, cache=cache))
print(json.dumps(out))
