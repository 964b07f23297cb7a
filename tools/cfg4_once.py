import sys, torch
sys.path.insert(0, '.')
import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import synthetic
trees = [synthetic.shell_tree(seed=s) for s in range(4)]
scene, cam = synthetic.scene_config4(trees)
for f in range(6):
    vv.render_scene(scene, cam, f, vv.RenderOptions(frame_slice="per_sample"), out="torch")
torch.cuda.synchronize()
