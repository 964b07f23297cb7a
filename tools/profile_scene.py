"""Driver for ncu: the cfg4 scene (4 performers, 1080p)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

trees = [synthetic.shell_tree(seed=s) for s in range(4)]
scene, cam = synthetic.scene_config4(trees)
for f in range(4):
    vv.render_scene(scene, cam, f, out="torch")
torch.cuda.synchronize()
print("ok")
