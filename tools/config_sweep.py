"""Time every BASELINE.json configuration on ONE GPU through the public API.

    python tools/config_sweep.py [--frames N]

cfg1 depth-7 64x64 (n_max 1), cfg2 depth-9 1080p sweep (n_max 2, T 30),
cfg3 motion tree 1080p (T 60), cfg4 four performers composed at 1080p,
cfg5 stereo 2 x 2160x2160 (both eyes on this one GPU; the 8-GPU tile path is
distributed.TileRenderer).  Device-resident outputs, CUDA events on the
current stream, per-frame slice pass included (what render() does).
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=10)
args = ap.parse_args()
dev = torch.device("cuda", 0)


def timed(fn, frames, warm=3):
    for f in range(warm):
        fn(f)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for f in range(frames):
        fn(f)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / frames


def single(tree, cam, nframes):
    h, w = cam.height, cam.width
    rgb = torch.empty((h, w, 3), device=dev)
    a = torch.empty((h, w), device=dev)
    d = torch.empty((h, w), device=dev)
    T = tree.frames
    return timed(lambda f: vv.render_into(tree, cam, f % T, rgb, a, d), nframes)


out = {}
c1 = synthetic.CONFIGS[1]
t1 = synthetic.shell_tree(depth=7, n_max=1, frames=16, seed=0)
ms = single(t1, synthetic.bench_camera(64, 64), args.frames)
out["cfg1"] = dict(ms=ms, mrays=64 * 64 / ms / 1e3)
t2 = synthetic.shell_tree()
cam = synthetic.bench_camera()
ms = single(t2, cam, args.frames)
out["cfg2"] = dict(ms=ms, mrays=cam.width * cam.height / ms / 1e3, fps=1e3 / ms)
t3 = synthetic.motion_tree()
ms = single(t3, cam, args.frames)
out["cfg3"] = dict(ms=ms, mrays=cam.width * cam.height / ms / 1e3, fps=1e3 / ms)
del t3
trees = [t2] + [synthetic.shell_tree(seed=s) for s in (1, 2, 3)]
scene, cam4 = synthetic.scene_config4(trees)
ms = timed(lambda f: vv.render_scene(scene, cam4, f, out="torch"), args.frames)
rays = 4 * cam4.width * cam4.height
out["cfg4"] = dict(ms=ms, mrays_pulled_back=rays / ms / 1e3, fps=1e3 / ms, instances=4)
eyes = synthetic.stereo_cameras()
h = w = eyes[0].width
bufs = [(torch.empty((h, w, 3), device=dev), torch.empty((h, w), device=dev), torch.empty((h, w), device=dev))
        for _ in eyes]


def stereo(f):  # one slice pass per frame, shared by both eyes
    cache = vv.build_frame_cache(t2, f % 30)
    for cam_e, (r, a, d) in zip(eyes, bufs):
        vv.render_into(t2, cam_e, f % 30, r, a, d, cache=cache)


ms = timed(stereo, args.frames)
out["cfg5_1gpu"] = dict(ms=ms, mrays=2 * h * w / ms / 1e3, fps=1e3 / ms)
print(json.dumps({k: {kk: round(vv_, 3) if isinstance(vv_, float) else vv_ for kk, vv_ in v.items()}
                  for k, v in out.items()}))
