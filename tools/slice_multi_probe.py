"""Slice passes: K single-frame passes vs one K-frame pass (cfg2)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

import os  # noqa: E402

tree = synthetic.motion_tree() if os.environ.get("VV_PROBE_TREE") == "motion" else synthetic.shell_tree()


def timed(fn, n=20):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(n):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


def group(i, k):  # a sweep of consecutive frames, like playback
    return [(3 + k * i + j) % tree.frames for j in range(k)]


for k in (1, 2, 3, 4):
    t1 = timed(lambda i: [vv.build_frame_cache(tree, f) for f in group(i, k)])
    tk = timed(lambda i: vv.build_frame_caches(tree, group(i, k)))
    print(f"K={k}: {k} single passes {t1:.3f} ms | one {k}-frame pass {tk:.3f} ms")
    tr = timed(lambda i: vv.build_frame_caches(tree, group(i, k), render_only=True))
    print(f"K={k}: one {k}-frame render-only pass {tr:.3f} ms")
