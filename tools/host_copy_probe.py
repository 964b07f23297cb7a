"""render() -> numpy at cfg2: banded device->host copies behind the render
(vv_render_camera_to_host) for several band heights, against the plain
render + one copy, and the copy alone."""
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
n = 5 * cam.width * cam.height
dev_buf = torch.empty(n, device="cuda")
host = torch.empty(n, pin_memory=True)


def wall(fn, k=20):
    for f in range(3):
        fn(f)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for f in range(k):
        fn(f % 30)
    torch.cuda.synchronize()
    return round((time.perf_counter() - t) / k * 1e3, 4)


def copy_only(f):
    host.copy_(dev_buf, non_blocking=True)


out = {"copy_only_ms": wall(copy_only)}
out["render_torch_ms"] = wall(lambda f: vv.render(tree, cam, f, out="torch"))
for rows in ("1080", "272", "136", "104", "64"):
    os.environ["VV_HOST_BAND_ROWS"] = rows
    out[f"render_numpy_bands{rows}_ms"] = wall(lambda f: vv.render(tree, cam, f))
print(out)
