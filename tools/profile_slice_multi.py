"""Driver for ncu: cfg2 slice passes, 1 and 4 frames per payload read."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

tree = synthetic.shell_tree()
for i in range(3):
    c = vv.build_frame_caches(tree, [0, 1, 2, 3])
    c1 = vv.build_frame_cache(tree, 4)
    del c, c1
torch.cuda.synchronize()
print("ok")
