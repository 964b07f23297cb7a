"""One bench step of a config after its warm-up steps, for ncu captures of
the dominant kernel (bench.py's Stepper: exactly the timed step's launches).

    ncu --set full -k regex:k_render_camera --launch-skip 3 -c 1 python tools/profile_step.py --config 2
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=4)
args = ap.parse_args()
dev = torch.device("cuda", 0)
wl = bench.Workload(args.config)
st = bench.Stepper(wl, dev)
frames = [(5 + i) % wl.frames_total for i in range(args.steps)]
st.prepare(frames)
for f in frames:
    st(f)
torch.cuda.synchronize()
print("PROFILE_STEP_OK", args.config, frames)
