"""Playback with the slice pass of frame f+1 on a second stream, concurrent
with the render of frame f: steady-state ms/frame vs the serial order."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

tree = synthetic.shell_tree()
cam = synthetic.bench_camera()
dev = torch.device("cuda", 0)
h, w = cam.height, cam.width
bufs = [(torch.empty((h, w, 3), device=dev), torch.empty((h, w), device=dev), torch.empty((h, w), device=dev))
        for _ in range(2)]
s_render = torch.cuda.Stream(dev)
s_slice = torch.cuda.Stream(dev, priority=-1)
N = 30


def serial():
    for f in range(N):
        with torch.cuda.stream(s_render):
            c = vv.build_frame_cache(tree, f % 30)
            r, a, d = bufs[f % 2]
            vv.render_into(tree, cam, f % 30, r, a, d, cache=c)
            del c


def pipelined():
    with torch.cuda.stream(s_slice):
        nxt = vv.build_frame_cache(tree, 0)
    ev = torch.cuda.Event()
    ev.record(s_slice)
    for f in range(N):
        cur, cur_ev = nxt, ev
        s_render.wait_event(cur_ev)
        if f + 1 < N:
            with torch.cuda.stream(s_slice):
                nxt = vv.build_frame_cache(tree, (f + 1) % 30)
            ev = torch.cuda.Event()
            ev.record(s_slice)
        with torch.cuda.stream(s_render):
            r, a, d = bufs[f % 2]
            vv.render_into(tree, cam, f % 30, r, a, d, cache=cur)
        done = torch.cuda.Event()
        done.record(s_render)
        s_slice.wait_event(done)  # the slice pool block of `cur` is freed on s_slice after its render
        del cur


for name, fn in (("serial", serial), ("pipelined", pipelined), ("serial", serial), ("pipelined", pipelined)):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()  # work runs on side streams: wall clock over a GPU-bound loop
    fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / N * 1e3:.3f} ms/frame")
