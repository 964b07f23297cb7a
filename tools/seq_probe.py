"""Where does render_sequence spend its time?  Per-yield wall times plus D2H bandwidth."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
frames = list(range(30))
R = sys.modules["paper_2202_06088_b200.render"]

_get = R._PINNED.get
_log = []


def timed_get(n):
    t = time.perf_counter()
    before = sum(len(v) for v in R._PINNED._free.values())
    r = _get(n)
    after = sum(len(v) for v in R._PINNED._free.values())
    _log.append((round((time.perf_counter() - t) * 1e3, 2), after - before))
    return r


R._PINNED.get = timed_get
_ri = R.render_into
_rlog = []


def timed_ri(*a, **k):
    t = time.perf_counter()
    r = _ri(*a, **k)
    _rlog.append(round((time.perf_counter() - t) * 1e3, 2))
    return r


R.render_into = timed_ri
for _ in vv.render_sequence(tree, cam, frames[:4]):
    pass
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    ts = []
    for layer in vv.render_sequence(tree, cam, frames):
        ts.append(time.perf_counter())
    t1 = time.perf_counter()
    d = [round((b - a) * 1e3, 2) for a, b in zip([t0] + ts[:-1], ts)]
    print("  pinned gets (ms, new):", _log[:6], " render_into ms:", _rlog[:4])
    _log.clear(); _rlog.clear()
    print(f"seq rep{rep}: {(t1 - t0) / len(frames) * 1e3:.3f} ms/frame; per-yield ms {d[:8]} ... {d[-4:]}")
h, w = cam.height, cam.width
buf = torch.empty(5 * h * w, dtype=torch.float32, device="cuda")
host = torch.empty(5 * h * w, dtype=torch.float32, pin_memory=True)
for _ in range(3):
    host.copy_(buf, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(10):
    host.copy_(buf, non_blocking=True)
    torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"D2H 41.5 MB pinned: {(t1 - t0) / 10 * 1e3:.3f} ms ({5 * h * w * 4 / ((t1 - t0) / 10) / 1e9:.1f} GB/s)")
s = torch.cuda.Stream()
t0 = time.perf_counter()
for i in range(10):
    with torch.cuda.stream(s):
        host.copy_(buf, non_blocking=True)
    s.synchronize()
t1 = time.perf_counter()
print(f"D2H side stream: {(t1 - t0) / 10 * 1e3:.3f} ms")
t0 = time.perf_counter()
for i in range(10):
    x = host.numpy().copy()
t1 = time.perf_counter()
print(f"host memcpy 41.5 MB: {(t1 - t0) / 10 * 1e3:.3f} ms")
t0 = time.perf_counter()
for i in range(10):
    layer = vv.render(tree, cam, i)
t1 = time.perf_counter()
print(f"render(): {(t1 - t0) / 10 * 1e3:.3f} ms")
