"""cfg3 (motion tree, 1080p, T 60): frame time with / without per-frame node
masks and with the regular / long segment queue, single-frame render and
4-frame shared-walk playback.

    python tools/cfg3_mask_probe.py [--frames N] [--config 2|3]
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

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=20)
ap.add_argument("--config", type=int, default=3)
args = ap.parse_args()
dev = torch.device("cuda", 0)
tree = synthetic.motion_tree() if args.config == 3 else synthetic.shell_tree()
cam = synthetic.bench_camera()
h, w = cam.height, cam.width
T = tree.frames
outs = [(torch.empty((h, w, 3), device=dev), torch.empty((h, w), device=dev), torch.empty((h, w), device=dev))
        for _ in range(4)]


def timed(fn, n, warm=3):
    for f in range(warm):
        fn(f)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for f in range(n):
        fn(f)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


def single(f):
    vv.render_into(tree, cam, (7 * f) % T, *outs[0])


def render_only(caches):
    def fn(f):
        vv.render_into(tree, cam, caches[f % len(caches)].frame, *outs[0], cache=caches[f % len(caches)])
    return fn


def playback(f):
    fr = [(4 * f + k) % T for k in range(4)]
    vv.render_frames_into(tree, cam, fr, outs)


res = {}
for mask in ("0", "1"):
    for lq in ("0", "1"):
        os.environ["VV_NODE_MASK"] = mask
        os.environ["VV_LONG_QUEUE"] = lq
        caches = [vv.build_frame_caches(tree, [f], render_only=True)[0] for f in range(0, T, T // 8)]
        torch.cuda.synchronize()
        res[f"mask{mask}_lq{lq}"] = dict(frame_ms=round(timed(single, args.frames), 4),
                                         render_kernel_ms=round(timed(render_only(caches), args.frames), 4),
                                         playback_ms_per_frame=round(timed(playback, args.frames // 4 or 1) / 4, 4))
        del caches
print(json.dumps({"config": args.config, **res}))
