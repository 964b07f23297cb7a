"""Visible-set slices at cfg2: set size, slice-pass and render-kernel times
with VV_SLICE_VISIBLE vs render-only slices (CUDA events, L2 flushed).

    python tools/visible_probe.py
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402
from paper_2202_06088_b200.device import replica  # noqa: E402

dev = torch.device("cuda", 0)
tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
rep = replica(tree, dev)
h, w = cam.height, cam.width
out = [torch.empty((h, w, 3), device=dev), torch.empty((h, w), device=dev), torch.empty((h, w), device=dev)]
flush = torch.empty(128 * 2**20, dtype=torch.float32, device=dev)
plan = vv.CameraPlan(dev)
res = {"n_leaves": tree.n_leaves}


def run(visible, n=24):
    sl, rd = [], []
    per = []
    for i in range(n):
        f = (7 * i) % 30
        flush.zero_()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        fs = vv.build_frame_caches(tree, [f], visible=visible, render_only=True)[0]
        b.record()
        vv.render_into(tree, cam, f, *out, cache=fs, plan=plan)
        c.record()
        torch.cuda.synchronize()
        if i >= 4:
            sl.append(a.elapsed_time(b))
            rd.append(b.elapsed_time(c))
            per.append((round(a.elapsed_time(b), 3), round(b.elapsed_time(c), 3)))
        del fs
    return {"slice_ms": round(sum(sl) / len(sl), 4), "render_ms": round(sum(rd) / len(rd), 4), "per_frame": per}


if os.environ.get("VV_PROBE_VIS_ONLY"):  # for an ncu launch list of the visible-set path alone
    run(True, 12)
    print(json.dumps({"visible_set": rep.visible_count()}))
    sys.exit(0)
res["render_only"] = run(False)
if not os.environ.get("VV_LIB_PATH") or os.environ.get("VV_PROBE_FORCE_VIS"):
    res["visible"] = run(True)
    res["visible_set"] = rep.visible_count()
    res["render_only_again"] = run(False)
print(json.dumps(res))
