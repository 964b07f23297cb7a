"""How much would compacting hit rays into dense warps save?"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
W, H = cam.width, cam.height
o, d = cam.rays()
# 8x4 chunk order (the camera kernel's warp layout)
ix, iy = np.meshgrid(np.arange(W), np.arange(H), indexing="xy")
key = ((iy // 4) * (W // 8) + (ix // 8)) * 32 + (iy % 4) * 8 + (ix % 8)
order = np.argsort(key.reshape(-1), kind="stable")
o, d = o[order], d[order]
dev = torch.device("cuda", 0)
ot, dt = torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev)
fs = vv.build_frame_cache(tree, 3)
p, a, t = vv.render_rays(tree, ot, dt, 3, cache=fs)
hit = (a > 0).cpu().numpy()
print("hit fraction", hit.mean())
sets = {"all": np.arange(len(o)), "hit": np.nonzero(hit)[0], "miss": np.nonzero(~hit)[0]}
for name, idx in sets.items():
    oo, dd = ot[torch.from_numpy(idx).to(dev)].contiguous(), dt[torch.from_numpy(idx).to(dev)].contiguous()
    for _ in range(2):
        vv.render_rays(tree, oo, dd, 3, cache=fs)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        vv.render_rays(tree, oo, dd, 3, cache=fs)
    e.record()
    torch.cuda.synchronize()
    print(f"{name:5s} rays {len(idx):8d}: {s.elapsed_time(e) / 5:.3f} ms")
