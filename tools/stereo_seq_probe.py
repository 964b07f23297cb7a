"""cfg5 end to end: both eyes' render_sequence zipped, repeated; per-pair
delivery times and pinned-pool state, to find where a slow run loses time.

    python tools/stereo_seq_probe.py
"""
import collections
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402
from paper_2202_06088_b200.render import _PINNED  # noqa: E402

tree = synthetic.shell_tree()
eyes = synthetic.stereo_cameras()
frames = [(3 + i) % 30 for i in range(30)]
for _ in range(2):
    collections.deque(zip(*[vv.render_sequence(tree, c, frames[:6]) for c in eyes]), maxlen=0)
torch.cuda.synchronize()
out = []
for rep in range(4):
    t0 = time.perf_counter()
    gaps = []
    last = t0
    for pair in zip(*[vv.render_sequence(tree, c, frames) for c in eyes]):
        now = time.perf_counter()
        gaps.append(round((now - last) * 1e3, 2))
        last = now
    tot = time.perf_counter() - t0
    pool = {k: len(v) for k, v in _PINNED._free.items()}
    out.append({"rep": rep, "ms_per_pair": round(tot / len(frames) * 1e3, 3), "max_gap": max(gaps),
                "slow_gaps": [g for g in gaps if g > 6], "pool": pool})
    print(json.dumps(out[-1]), flush=True)
