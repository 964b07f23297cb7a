"""Camera-kernel time with and without chunk-box coverage (VV_COVERAGE),
cfg2 / cfg3 at 1080p from a prebuilt render-only slice, L2 flushed; plans on
and off.  Also the coverage fraction of the frame."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

out = {}
flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")
for name, tree in (("cfg2", synthetic.shell_tree()), ("cfg3", synthetic.motion_tree())):
    cam = synthetic.bench_camera()
    h, w = cam.height, cam.width
    o = (torch.empty((h, w, 3), device="cuda"), torch.empty((h, w), device="cuda"), torch.empty((h, w), device="cuda"))
    caches = [vv.build_frame_caches(tree, [f], render_only=True)[0] for f in (3, 11, 19, 27)]

    def ev(fn, n=12):
        for i in range(4):
            fn(i)
        tot = 0.0
        for i in range(n):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn(i)
            e.record()
            torch.cuda.synchronize()
            tot += s.elapsed_time(e)
        return round(tot / n, 4)

    for cov in ("0", "1"):
        os.environ["VV_COVERAGE"] = cov
        plan = vv.CameraPlan()
        out[f"{name}_cov{cov}_static"] = ev(lambda i: vv.render_into(tree, cam, caches[i % 4].frame, *o,
                                                                     cache=caches[i % 4]))
        out[f"{name}_cov{cov}_plan"] = ev(lambda i: vv.render_into(tree, cam, caches[i % 4].frame, *o,
                                                                   cache=caches[i % 4], plan=plan))
    os.environ.pop("VV_COVERAGE")
print(json.dumps(out))
