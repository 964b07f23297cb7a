import sys, torch
sys.path.insert(0, '.')
import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import synthetic
trees = [synthetic.shell_tree(seed=s) for s in range(4)]
scene, cam = synthetic.scene_config4(trees)
def timed(fn, n=10):
    for f in range(3): fn(f)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for f in range(n): fn(f)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
for mode in ("auto", "per_sample", "per_frame"):
    o = vv.RenderOptions(frame_slice=mode)
    print(mode, round(timed(lambda f: vv.render_scene(scene, cam, f, o, out="torch")), 3), "ms")
a = vv.render_scene(scene, cam, 4, vv.RenderOptions(frame_slice="per_sample"), out="torch")
b = vv.render_scene(scene, cam, 4, vv.RenderOptions(frame_slice="per_frame"), out="torch")
print("bitwise equal:", torch.equal(a, b))
