"""render_sequence end to end (numpy frames on the host) for 30 cfg2
frames, with SEQUENCE_GROUP = 2, 3, 4 (frames per shared walk)."""
import collections
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

R = sys.modules["paper_2202_06088_b200.render"]
tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
n_rays = cam.width * cam.height
for _ in range(2):
    collections.deque(vv.render_sequence(tree, cam, range(8)), maxlen=0)
torch.cuda.synchronize()
for rep in range(3):
    row = {}
    for g in (2, 3, 4):
        R.SEQUENCE_GROUP = g
        collections.deque(vv.render_sequence(tree, cam, range(8)), maxlen=0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for layer in vv.render_sequence(tree, cam, range(30)):
            pass
        row[g] = round(30 * n_rays / (time.perf_counter() - t) / 1e6, 1)
    print("Mrays/s by group:", row, flush=True)
