"""Per-frame traversal statistics of the config-2 bench frame on the GPU:
visited / distinct leaves, hit fraction, per-ray P/V/S (reference-defined)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
tree = synthetic.motion_tree() if cfg == 3 else synthetic.shell_tree()
cam = synthetic.bench_camera(1920, 1080)
o, d = cam.rays()
for frame in (3, 15):
    t0 = time.time()
    used, start, leaf = vv.render_ray_visits(tree, o, d, frame)
    p, a, t, st = vv.render_rays(tree, o, d, frame, stats=True)
    uniq = np.unique(leaf)
    print(f"cfg{cfg} frame {frame}: rays {len(used)}, hit {np.mean(a > 0):.3f}, visits {len(leaf)}, "
          f"distinct leaves {len(uniq)} of {tree.n_leaves} ({len(uniq) / tree.n_leaves:.3f}), "
          f"visits/distinct {len(leaf) / max(1, len(uniq)):.2f}, P {st['node_pops'].mean():.2f} "
          f"V {st['sample_count'].mean():.2f} S {st['shaded'].mean():.2f} ({time.time() - t0:.1f}s)")
