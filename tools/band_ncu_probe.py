"""Full-frame render kernel, then one 96-row band (rows 552-648) of the same
frame from the same cache, both with persistent warps in cost order
(VV_CAM_QUEUE=1 + block_order): for an ncu --set full comparison of a short
region kernel against the full frame."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402
from paper_2202_06088_b200.distributed import block_order, render_region  # noqa: E402

tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
h, w = cam.height, cam.width
rgb = torch.empty((h, w, 3), device="cuda")
alpha = torch.empty((h, w), device="cuda")
depth = torch.empty((h, w), device="cuda")
used = torch.empty((h, w), dtype=torch.int32, device="cuda")
cache = vv.build_frame_cache(tree, 5)
vv.render_into(tree, cam, 0, rgb, alpha, depth, sample_count=used)  # cost map (kernel 1)
costs = used.to(torch.float64) + 1.0
os.environ["VV_CAM_QUEUE"] = "1"
render_region(tree, cam, 5, (0, 0, w, h), rgb, alpha, depth, cache=cache, order=block_order(costs, (0, 0, w, h)))
render_region(tree, cam, 5, (0, 552, w, 648), rgb, alpha, depth, cache=cache,
              order=block_order(costs, (0, 552, w, 648)))
torch.cuda.synchronize()
