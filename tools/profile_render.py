"""Short driver for ncu: build the config-2 tree, render a few 1080p frames.

    python tools/profile_render.py [--frames N] [--cached] [--config 2|3]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=4)
ap.add_argument("--cached", action="store_true")
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--size", default="1920x1080")
args = ap.parse_args()
w, h = (int(v) for v in args.size.split("x"))
tree = synthetic.motion_tree() if args.config == 3 else synthetic.shell_tree()
cam = synthetic.bench_camera(w, h)
dev = torch.device("cuda", 0)
rgb = torch.empty((h, w, 3), device=dev)
alpha = torch.empty((h, w), device=dev)
depth = torch.empty((h, w), device=dev)
times = []
for f in range(args.frames):
    cache = vv.build_frame_cache(tree, f) if args.cached else None
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    vv.render_into(tree, cam, f, rgb, alpha, depth, cache=cache)
    e.record()
    torch.cuda.synchronize()
    times.append(s.elapsed_time(e))
print("frame ms:", " ".join(f"{t:.3f}" for t in times))
