"""cfg2 .voct (1.5 GB) -> device: host VOctree.load + upload vs load_device."""
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402
from paper_2202_06088_b200.device import replica  # noqa: E402

tree = synthetic.shell_tree()
path = os.path.join(tempfile.gettempdir(), "vv_cfg2.voct")
tree.save(path)
del tree
torch.cuda.init()
for rep in range(2):
    t0 = time.perf_counter()
    host = vv.VOctree.load(path)
    t1 = time.perf_counter()
    replica(host)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del host
    t3 = time.perf_counter()
    dev = vv.load_device(path)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"rep {rep}: VOctree.load {t1 - t0:.2f}s + upload {t2 - t1:.2f}s = {t2 - t0:.2f}s | "
          f"load_device {t4 - t3:.2f}s ({os.path.getsize(path) / 1e9:.2f} GB)")
    del dev
