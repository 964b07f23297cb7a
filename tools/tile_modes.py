"""One rank's share of a tile-sharded cfg2 frame (1/world of the 64x64 tiles):
per-frame slice pass vs per-sample decode vs the auto choice."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402
from paper_2202_06088_b200.distributed import TileRenderer  # noqa: E402

import os  # noqa: E402

tree = synthetic.motion_tree() if os.environ.get("VV_PROBE_TREE") == "motion" else synthetic.shell_tree()
cam = synthetic.bench_camera()


def timed(fn, n=10):
    for f in range(3):
        fn(f)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for f in range(n):
        fn(f)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


for world in (1, 2, 3, 4, 6, 8):
    tr = TileRenderer(cam.width, cam.height, 64, rank=0, world=world)
    row = []
    for mode in ("auto", "per_frame", "per_sample"):
        o = vv.RenderOptions(frame_slice=mode)
        row.append(f"{mode} {timed(lambda f: tr.render_slab(tree, cam, f % tree.frames, o)):.3f} ms")
    print(f"world {world}: " + " | ".join(row))
