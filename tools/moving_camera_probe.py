"""cfg2 tree, 1080p, a camera orbiting the shell (STEP degrees of azimuth per
frame): per-frame device time of render_into (stream plan) with the visible
set on and off -- the set follows a moving view through its misses and
census frames; this measures what that costs against a fixed camera.

    VV_VISIBLE=0|1 python tools/moving_camera_probe.py [step_deg]
"""
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

step = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
tree = synthetic.shell_tree()
c = np.asarray(tree.bbox_lo) + 0.5 * tree.side
eye0 = np.array([1.6, 1.3, 0.9])
r = np.linalg.norm((eye0 - c)[:2])
z = eye0[2]
a0 = math.atan2(eye0[1] - c[1], eye0[0] - c[0])


def cam(i):
    a = a0 + math.radians(step * i)
    return vv.Camera.look_at([c[0] + r * math.cos(a), c[1] + r * math.sin(a), z], (0.5, 0.5, 0.5),
                             up=(0.0, 0.0, 1.0), width=1920, height=1080, focal=1.08 * 1920)


dev = torch.device("cuda", 0)
out = [torch.empty((1080, 1920, 3), device=dev), torch.empty((1080, 1920), device=dev),
       torch.empty((1080, 1920), device=dev)]
plan = vv.CameraPlan(dev)
flush = torch.empty(128 * 2**20, dtype=torch.float32, device=dev)
for i in range(8):
    vv.render_into(tree, cam(i), i % 30, *out, plan=plan)
torch.cuda.synchronize()
ts = []
for i in range(8, 68):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    vv.render_into(tree, cam(i), i % 30, *out, plan=plan)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
print(json.dumps({"visible": os.environ.get("VV_VISIBLE", "default"), "step_deg": step,
                  "mean_ms": round(sum(ts) / len(ts), 4), "max_ms": round(max(ts), 4),
                  "first10": [round(t, 3) for t in ts[:10]]}))
