"""A/B: frame_slice "per_frame" (slice pass + one-pass render kernel) vs
"deferred" (sigma slice, weight walk, colour of the shaded leaves, colour
pass) through render_into, cfg2 and cfg3, frame sweep, L2 flushed between
frames (outside the events)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

dev = torch.device("cuda", 0)
cam = synthetic.bench_camera()
rgb = torch.empty((cam.height, cam.width, 3), device=dev)
a = torch.empty((cam.height, cam.width), device=dev)
d = torch.empty((cam.height, cam.width), device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def run(tree, mode, frames=20):
    opts = vv.RenderOptions(frame_slice=mode)
    for f in range(4):
        vv.render_into(tree, cam, f % tree.frames, rgb, a, d, opts)
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(frames):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        vv.render_into(tree, cam, (3 + i) % tree.frames, rgb, a, d, opts)
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / frames


for name, tree in (("cfg2", synthetic.shell_tree()), ("cfg3", synthetic.motion_tree())):
    for _ in range(2):
        print(name, {m: round(run(tree, m), 4) for m in ("per_frame", "deferred")}, flush=True)
