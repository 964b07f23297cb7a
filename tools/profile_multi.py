"""Driver for ncu: cfg2 playback groups (4 frames per walk, as bench.py's playback)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
outs = [(torch.empty((1080, 1920, 3), device="cuda"), torch.empty((1080, 1920), device="cuda"),
         torch.empty((1080, 1920), device="cuda")) for _ in range(4)]
for g in range(4):
    vv.render_frames_into(tree, cam, [4 * g + k for k in range(4)], outs)
torch.cuda.synchronize()
print("ok")
