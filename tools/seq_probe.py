"""render_sequence (playback to numpy) at cfg2: per-frame wall time for
sequence lengths 20 / 40 / 80 and first-group sizes 0 (groups of 3 from the
start) / 1 / 2, plus the steady-state per-frame cost (80 - 40 frames)."""
import collections
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
for _ in range(2):
    collections.deque(vv.render_sequence(tree, cam, list(range(6))), maxlen=0)
torch.cuda.synchronize()
out = {}
for first in ("0", "1", "2"):
    os.environ["VV_SEQ_FIRST"] = first
    for n in (20, 40, 80):
        frames = [(5 + i) % 30 for i in range(n)]
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            collections.deque(vv.render_sequence(tree, cam, frames), maxlen=0)
            ts.append(time.perf_counter() - t)
        out[f"first{first}_n{n}_ms_per_frame"] = round(min(ts) / n * 1e3, 4)
    out[f"first{first}_steady_ms"] = round((out[f"first{first}_n80_ms_per_frame"] * 80
                                            - out[f"first{first}_n40_ms_per_frame"] * 40) / 40, 4)
print(json.dumps(out))
