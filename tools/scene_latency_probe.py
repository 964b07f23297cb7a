"""Per-call latency of compose.render_scene (cfg4 scene) -> numpy and -> torch,
with a cProfile of the numpy path: where does a call's host time go?

    python tools/scene_latency_probe.py
"""
import cProfile
import io
import json
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from bench import Workload  # noqa: E402

wl = Workload(4)
dev = torch.device("cuda", 0)
cam = wl.cams[0]
for f in range(6):
    vv.render_scene(wl.scene, cam, f)
torch.cuda.synchronize()
out = {}
for kind in ("torch", "numpy"):
    ts = []
    for f in range(40):
        t = time.perf_counter()
        img = vv.render_scene(wl.scene, cam, f % 30, out=kind)
        if kind == "torch":
            torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    ts.sort()
    out[kind] = {"median_ms": round(ts[len(ts) // 2], 3), "mean_ms": round(sum(ts) / len(ts), 3),
                 "min_ms": round(ts[0], 3), "max_ms": round(ts[-1], 3)}
t = time.perf_counter()
for f in range(20):
    vv.render_scene(wl.scene, cam, f, out="torch")
torch.cuda.synchronize()
out["torch_async_ms_per_call"] = round((time.perf_counter() - t) / 20 * 1e3, 3)
pr = cProfile.Profile()
pr.enable()
for f in range(20):
    vv.render_scene(wl.scene, cam, f)
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25)
print(s.getvalue(), file=sys.stderr)
print(json.dumps(out))
