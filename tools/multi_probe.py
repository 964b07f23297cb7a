"""Two frames of one camera in one walk (vv_render_camera_multi) vs two
single-frame renders: bitwise comparison and timing (cfg2 / cfg3)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import _native, synthetic  # noqa: E402
from paper_2202_06088_b200.device import replica, stream_ptr  # noqa: E402

dev = torch.device("cuda", 0)


def run(tree, name, KF=2):
    cam = synthetic.bench_camera()
    h, w = cam.height, cam.width
    rep = replica(tree, dev)
    outs = [[torch.empty((h, w, 3), device=dev), torch.empty((h, w), device=dev), torch.empty((h, w), device=dev)]
            for _ in range(KF)]
    refs = [[torch.empty((h, w, 3), device=dev), torch.empty((h, w), device=dev), torch.empty((h, w), device=dev)]
            for _ in range(KF)]
    oc = vv.RenderOptions().c_struct()
    cd = cam.desc()
    P = ctypes.c_void_p

    def multi(f0, caches):
        frames = (ctypes.c_int32 * KF)(*[f0 + k for k in range(KF)])
        cs = (P * KF)(*[c._handle for c in caches])
        rgb = (P * KF)(*[o[0].data_ptr() for o in outs])
        al = (P * KF)(*[o[1].data_ptr() for o in outs])
        de = (P * KF)(*[o[2].data_ptr() for o in outs])
        _native.check(_native.lib().vv_render_camera_multi(rep.handle, KF, frames, cs, ctypes.byref(oc),
                                                           ctypes.byref(cd), rgb, al, de, stream_ptr(dev)))

    T = tree.frames
    caches = {f: vv.build_frame_cache(tree, f) for f in range(8)}
    for f0 in (0, 4):
        multi(f0, [caches[f0 + k] for k in range(KF)])
        for k in range(KF):
            vv.render_into(tree, cam, f0 + k, *refs[k], cache=caches[f0 + k])
        torch.cuda.synchronize()
        same = all(torch.equal(a, b) for k in range(KF) for a, b in zip(outs[k], refs[k]))
        print(f"{name} K={KF} frames from {f0}: bitwise equal {same}")

    def timed(fn, n=10):
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i in range(n):
            fn(i)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / n

    t_multi = timed(lambda i: multi(4 * (i % 2), [caches[4 * (i % 2) + k] for k in range(KF)]))
    t_single = timed(lambda i: [vv.render_into(tree, cam, 4 * (i % 2) + k, *refs[k], cache=caches[4 * (i % 2) + k])
                                for k in range(KF)])
    print(f"{name}: {KF} frames in one walk {t_multi:.3f} ms vs {KF} renders {t_single:.3f} ms "
          f"({t_single / t_multi:.2f}x on the render kernels, {t_multi / KF:.3f} ms per frame)")


t2 = synthetic.shell_tree()
for kf in (2, 3, 4):
    run(t2, "cfg2", kf)
del t2
t3 = synthetic.motion_tree()
for kf in (2, 3, 4):
    run(t3, "cfg3", kf)
