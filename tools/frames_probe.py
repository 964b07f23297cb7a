"""render_frames_into (slice pass for the group + one shared walk) per group size, cfg2."""
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
for k in (1, 2, 3, 4, 3, 4):
    def fn(i):
        vv.render_frames_into(tree, cam, [(4 * i + j) % 30 for j in range(k)], outs[:k])
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(8):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 8
    print(f"{k} frames: {ms:.3f} ms per group, {ms / k:.3f} ms per frame")
