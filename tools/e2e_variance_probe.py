"""Spread of the bench's end-to-end measurement (render_sequence of 20
cfg2 frames to numpy) over repeated runs on one box, after the same warm-up
the bench does."""
import collections
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
for f in range(3):
    vv.render(tree, cam, f)
for f in range(10):
    layer = vv.render(tree, cam, f)
del layer
for _ in range(2):
    collections.deque(vv.render_sequence(tree, cam, [0, 1, 2] * 2), maxlen=0)
torch.cuda.synchronize()
ms = []
for rep in range(12):
    frames = [(5 + i) % 30 for i in range(20)]
    t = time.perf_counter()
    for layer in vv.render_sequence(tree, cam, frames):
        pass
    ms.append((time.perf_counter() - t) / 20 * 1e3)
    del layer
print(json.dumps({"ms_per_frame": [round(x, 4) for x in ms], "median": round(statistics.median(ms), 4),
                  "min": round(min(ms), 4), "max": round(max(ms), 4)}))
