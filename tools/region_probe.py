"""One frame split into N row bands, every band rendered in turn on this GPU.

Default: launch list for ncu (--metrics gpu__time_duration.sum) -- chunk
culling, list-mode slice pass, render per band.  --timing: CUDA-event times
of the band render kernels alone (a full-frame slice passed as the cache)
against the full-frame render kernel, to separate the walk's own cost of a
band from its share of the decode.

    python tools/region_probe.py [--world 8] [--tree shell|motion] [--miss-cost 1.2] [--timing]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402
from paper_2202_06088_b200.distributed import band_plan, block_order, pixel_costs, render_region  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--tree", default="shell")
ap.add_argument("--miss-cost", type=float, default=1.0)
ap.add_argument("--timing", action="store_true")
args = ap.parse_args()
tree = synthetic.motion_tree() if args.tree == "motion" else synthetic.shell_tree()
cam = synthetic.bench_camera()
h, w = cam.height, cam.width
rgb = torch.empty((h, w, 3), device="cuda")
alpha = torch.empty((h, w), device="cuda")
depth = torch.empty((h, w), device="cuda")
costs = pixel_costs(tree, cam, 0, miss_cost=args.miss_cost)
edges = band_plan(costs.sum(dim=1).cpu().numpy(), args.world)
orders = [block_order(costs, (0, edges[r], w, edges[r + 1])) for r in range(args.world)]
print("edges", edges, file=sys.stderr, flush=True)
torch.cuda.synchronize()
if not args.timing:
    for r in range(args.world):
        render_region(tree, cam, 5, (0, edges[r], w, edges[r + 1]), rgb, alpha, depth, order=orders[r])
    torch.cuda.synchronize()
    sys.exit(0)

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
    return tot / n


full = ev(lambda: vv.render_into(tree, cam, 5, rgb, alpha, depth, cache=cache))
bands = [ev(lambda r=r: render_region(tree, cam, 5, (0, edges[r], w, edges[r + 1]), rgb, alpha, depth, cache=cache))
         for r in range(args.world)]
ordered = [ev(lambda r=r: render_region(tree, cam, 5, (0, edges[r], w, edges[r + 1]), rgb, alpha, depth, cache=cache,
                                        order=orders[r])) for r in range(args.world)]
full_order = block_order(costs, (0, 0, w, h))
full_ordered = ev(lambda: render_region(tree, cam, 5, (0, 0, w, h), rgb, alpha, depth, cache=cache, order=full_order))
print(json.dumps({"world": args.world, "edges": edges, "full_render_ms": round(full, 4),
                  "full_ordered_ms": round(full_ordered, 4),
                  "band_render_ms": [round(b, 4) for b in bands], "sum": round(sum(bands), 4),
                  "band_ordered_ms": [round(b, 4) for b in ordered], "sum_ordered": round(sum(ordered), 4)}))
