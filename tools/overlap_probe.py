"""Does frame rendering overlap with device->host copies?"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
h, w = cam.height, cam.width
n = 5 * h * w
dev = torch.device("cuda", 0)
buf = torch.empty(n, device=dev)
host = torch.empty(n, pin_memory=True)
rgb, al, de = buf[: 3 * h * w].view(h, w, 3), buf[3 * h * w: 4 * h * w].view(h, w), buf[4 * h * w:].view(h, w)
for i in range(3):
    vv.render_into(tree, cam, i, rgb, al, de)
torch.cuda.synchronize()
K = 20
t0 = time.perf_counter()
for i in range(K):
    vv.render_into(tree, cam, i % 30, rgb, al, de)
torch.cuda.synchronize()
print(f"render only: {(time.perf_counter() - t0) / K * 1e3:.3f} ms/frame")
t0 = time.perf_counter()
for i in range(K):
    vv.render_into(tree, cam, i % 30, rgb, al, de)
enq = (time.perf_counter() - t0) / K * 1e3
torch.cuda.synchronize()
print(f"enqueue cost: {enq:.3f} ms/frame")
cs = torch.cuda.Stream()
t0 = time.perf_counter()
for i in range(K):
    with torch.cuda.stream(cs):
        host.copy_(buf, non_blocking=True)
torch.cuda.synchronize()
print(f"copy only: {(time.perf_counter() - t0) / K * 1e3:.3f} ms/frame")
rs = torch.cuda.Stream()
t0 = time.perf_counter()
for i in range(K):
    with torch.cuda.stream(rs):
        vv.render_into(tree, cam, i % 30, rgb, al, de)
    with torch.cuda.stream(cs):
        host.copy_(buf, non_blocking=True)
torch.cuda.synchronize()
print(f"render(stream A) + copy(stream B) unordered: {(time.perf_counter() - t0) / K * 1e3:.3f} ms/frame")
for l in vv.render_sequence(tree, cam, [0, 1, 2]):
    pass
for rep in range(2):
    t0 = time.perf_counter()
    for l in vv.render_sequence(tree, cam, [i % 30 for i in range(K)]):
        pass
    print(f"render_sequence: {(time.perf_counter() - t0) / K * 1e3:.3f} ms/frame")
print("default stream", torch.cuda.current_stream(), "flags nonblocking?", cs)
