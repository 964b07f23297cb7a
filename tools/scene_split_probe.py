"""cfg4: the fused scene kernel vs each rigid performer rendered alone
through the camera kernel with its pulled-back camera (device outputs),
to size a layer-per-instance + blend design."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402
from paper_2202_06088_b200.render import Camera  # noqa: E402

trees = [synthetic.shell_tree(seed=s) for s in range(4)]
scene, cam = synthetic.scene_config4(trees)
dev = torch.device("cuda", 0)
rgb = torch.empty((cam.height, cam.width, 3), device=dev)
a = torch.empty((cam.height, cam.width), device=dev)
d = torch.empty_like(a)


def timed(fn, n=10):
    for f in range(3):
        fn(f)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for f in range(n):
        fn(f)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


print("fused render_scene", round(timed(lambda f: vv.render_scene(scene, cam, f, out="torch")), 3), "ms")
for i, inst in enumerate(scene.instances):
    inv = np.linalg.inv(inst.effective_affine(0))
    m = inv @ cam.c2w
    R = m[:3, :3]
    if not np.allclose(R.T @ R, np.eye(3), atol=1e-9):
        print(f"instance {i}: not rigid (scaled), skipped")
        continue
    cam2 = Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, m)
    for mode in ("per_sample", "auto"):
        o = vv.RenderOptions(frame_slice=mode)
        t = timed(lambda f: vv.render_into(inst.tree, cam2, inst.local_frame(f), rgb, a, d, o))
        print(f"instance {i} alone, {mode}: {t:.3f} ms")
