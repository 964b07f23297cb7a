"""Whole-frame time (slice pass included) of the sliced and per-sample decode
paths through a camera plan, cfg2 / cfg3 / cfg5-eye, L2 flushed."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")
out = {}
shell = synthetic.shell_tree()
for name, tree, cam in (("cfg2", shell, synthetic.bench_camera()), ("cfg3", synthetic.motion_tree(), synthetic.bench_camera()),
                        ("cfg5_eye", shell, synthetic.stereo_cameras()[0])):
    h, w = cam.height, cam.width
    o = (torch.empty((h, w, 3), device="cuda"), torch.empty((h, w), device="cuda"), torch.empty((h, w), device="cuda"))
    for mode in ("per_frame", "per_sample"):
        plan = vv.CameraPlan()
        opts = vv.RenderOptions(frame_slice=mode)
        T = tree.frames

        def fn(i):
            vv.render_into(tree, cam, (3 * i) % T, *o, opts, plan=plan)
        for i in range(5):
            fn(i)
        tot = 0.0
        for i in range(12):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn(i)
            e.record()
            torch.cuda.synchronize()
            tot += s.elapsed_time(e)
        out[f"{name}_{mode}_ms"] = round(tot / 12, 4)
print(json.dumps(out))
