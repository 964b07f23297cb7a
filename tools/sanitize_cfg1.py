"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): config 1 (depth-7 shell, n_max 1, 64x64) through every kernel
family -- slice pass (1 and 4 frames, render-only with dark chunks), camera
kernel (static, persistent-warp plan, banded host copies), shared-walk
playback, node masks, region culling + list-mode slice, scene (Alg. 1,
lean and sliced) and joint composition, traversal queries.

    compute-sanitizer --tool memcheck python tools/sanitize_cfg1.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402
from paper_2202_06088_b200.distributed import band_plan, pixel_costs, render_region  # noqa: E402

tree = synthetic.shell_tree(depth=7, n_max=1, frames=16, seed=0)
motion = synthetic.motion_tree(depth=6, n_max=1, frames=12, seed=1)
cam = synthetic.bench_camera(64, 64)
h, w = cam.height, cam.width
dev = torch.device("cuda", 0)
outs = [(torch.empty((h, w, 3), device=dev), torch.empty((h, w), device=dev), torch.empty((h, w), device=dev))
        for _ in range(4)]

vv.render(tree, cam, 5)                                         # slice + camera + banded host copies
vv.render(tree, cam, 6, vv.RenderOptions(frame_slice="per_sample"))
plan = vv.CameraPlan(dev)
for f in (1, 2, 3):
    vv.render_into(tree, cam, f, *outs[0], plan=plan)           # persistent warps + plan order
vv.render_frames_into(tree, cam, [0, 3, 7, 9], outs)            # 4-frame slice + shared walk
os.environ["VV_NODE_MASK"] = "1"
vv.render(motion, cam, 4)                                       # dark chunks + node masks
vv.render_frames_into(motion, cam, [1, 2], outs[:2])
costs = pixel_costs(tree, cam, 0)
edges = band_plan(costs.sum(dim=1).cpu().numpy(), 3)
for r in range(3):                                              # chunk culling + list-mode slice
    render_region(motion, cam, 5, (0, edges[r], w, edges[r + 1]), *outs[1])
del os.environ["VV_NODE_MASK"]
o, d = cam.rays()
vv.render_ray_visits(tree, o[:512], d[:512], 5)                 # stats + visits kernels
vv.collect_segments(tree, o[:256], d[:256])
inst = [vv.SceneInstance(name="a", tree=tree),
        vv.SceneInstance(name="b", tree=tree, affine=np.diag([0.8, 0.8, 0.8, 1.0]),
                         timemap=vv.TimeMap.parse("shift(2)"))]
scene = vv.Scene(instances=inst)
vv.render_scene(scene, cam, 3)                                  # lean scene kernel
vv.render_scene(scene, cam, 3, vv.RenderOptions(frame_slice="per_frame"))
vv.render_scene(scene, cam, 3, mode="joint")                    # joint composition
torch.cuda.synchronize()
print("SANITIZE_WORKLOAD_OK")
