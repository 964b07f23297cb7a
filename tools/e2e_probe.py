"""Break down the public render() call (host-visible latency) on the GPU."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
for i in range(3):
    vv.render(tree, cam, i)
torch.cuda.synchronize()
n = 10
t0 = time.perf_counter()
for i in range(n):
    layer = vv.render(tree, cam, i % 30)
t1 = time.perf_counter()
print(f"render() -> numpy: {(t1 - t0) / n * 1e3:.3f} ms/frame")
t0 = time.perf_counter()
for i in range(n):
    layer = vv.render(tree, cam, i % 30, out="torch")
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"render(out=torch): {(t1 - t0) / n * 1e3:.3f} ms/frame")
h, w = cam.height, cam.width
buf = torch.empty(5 * h * w, dtype=torch.float32, device="cuda")
t0 = time.perf_counter()
for i in range(n):
    host = torch.empty(5 * h * w, dtype=torch.float32, pin_memory=True)
t1 = time.perf_counter()
print(f"pinned alloc: {(t1 - t0) / n * 1e3:.3f} ms")
host = torch.empty(5 * h * w, dtype=torch.float32, pin_memory=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    host.copy_(buf, non_blocking=True)
    torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"D2H 41.5 MB pinned: {(t1 - t0) / n * 1e3:.3f} ms ({5 * h * w * 4 / ((t1 - t0) / n) / 1e9:.1f} GB/s)")
